// ddks_kd.cuh — host side of the kd-ordered count (bit elision, DESIGN.md §7 "kd ordering"): reorder the packed
// rows label-major and hierarchically by x_0 .. x_{K-1} (K stable radix sorts), build the per-tile boxes, count with
// k_count<D, SPLIT, GT, K>. Instantiated per d in ddks_api_kd_*.cu (parallel compilation).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "ddks_kernels.cuh"
#include "ddks_kd_cluster.cuh"
#include "ddks_internal.h"
#include "ddks_launch.cuh"

namespace ddks_host {

struct KdChoice {
    int K;
    int64_t G0, G1, G2, G3;
};

#ifndef DDKS_KD_MAX  // deepest kd level instantiated: 4 (-DDDKS_KD_MAX=5 builds the 5-level variant, which measured
#define DDKS_KD_MAX 4  // slower: C5 755 vs 709 ms, d = 6 / 8 at N = 4e5 +15 % / +10 %)
#endif

inline int64_t lcm_i64(int64_t a, int64_t b) { return a / (int64_t)gcd_u64((uint64_t)a, (uint64_t)b) * b; }
inline int bits_for(uint64_t v) { int b = 0; while (v) { ++b; v >>= 1; } return b; }  // bits to hold 0..v

// Levels and cuts from a cost model of the compares per pair: D - K compared dims always, plus the expected
// undecided bits: a tile in the same slab (or, across labels, the neighbouring one) leaves bit 0 open
// (~1.0 / G0, fitted), bit 1 (~1.5 / G1), and the last sorted dim interleaves for (origins per CTA + TILE) /
// cell rows of the tiles (per warp for the last dim). Cells must keep at least A rows on average. forced_k (1..3) fixes K (tests); kmax caps it.
inline KdChoice kd_choose(int D, int64_t n_lab, int64_t RT, int64_t RW, int64_t TILE, int64_t A, int forced_k,
                          int kmax) {
    // tuning override DDKS_KD = "K[,G0[,G1[,G2]]]": K replaces the forced level; cuts not given come from the model
    int env_k = 0, env_n = 0;
    long long env_g[4] = {0, 0, 0, 0};
    if (const char* e = getenv("DDKS_KD")) {
        env_n = sscanf(e, "%d,%lld,%lld,%lld,%lld", &env_k, &env_g[0], &env_g[1], &env_g[2], &env_g[3]);
        if (env_n >= 1 && env_k >= 1 && env_k <= std::min(DDKS_KD_MAX, std::min(D, kmax))) forced_k = env_k;
        else env_n = 0;
    }
    KdChoice best{1, 1, 1, 1, 1};
    double best_cost = 1e300;
    // the last sorted dim is decided per warp: its open fraction scales with the warp's RW origins, not the CTA's RT
    (void)RT;
    const double c = (double)(RW + TILE) / (double)std::max<int64_t>(n_lab, 1);
    const int kcap = std::min(DDKS_KD_MAX, std::min(D, kmax));
    for (int K = 1; K <= kcap; ++K) {
        if (forced_k && K != forced_k) continue;
        const int64_t m0 = K >= 2 ? (K >= 3 ? 64 : 256) : 1, m1 = K >= 3 ? 64 : 1, m2 = K >= 4 ? 32 : 1,
                      m3 = K >= 5 ? 16 : 1;
        // K = 5 keeps only the loop variants with <= 2 open dims (kd_max_open): tiles with more run all 5 compares
        const double k5 = K >= 5 ? 0.1 : 0.0;
        for (int64_t g0 = 1; g0 <= m0; ++g0)
            for (int64_t g1 = 1; g1 <= m1; ++g1)
                for (int64_t g2 = 1; g2 <= m2; ++g2)
                    for (int64_t g3 = 1; g3 <= m3; ++g3) {
                        const int64_t cells = g0 * g1 * g2 * g3;
                        if (cells > 1 && n_lab / cells < A) break;  // a cell holds >= one origin block on average
                        double cost = (double)(D - K) + c * (double)cells + k5;
                        // level 0 weighs 1.0, not 1.5 (round 2, with the one-dim register path: C5 picks 6 x 9 x 9
                        // instead of 7 x 8 x 8, 630.9 -> 622 ms count; N = 4e5 at d = 5..8 within +-0.7 %;
                        // profiles/r2_kd_cuts_c5.txt, r2_kd_level0_weight.txt)
                        if (K >= 2) cost += 1.0 / (double)g0;
                        if (K >= 3) cost += 1.5 / (double)g1;
                        if (K >= 4) cost += 1.5 / (double)g2;
                        if (K >= 5) cost += 1.5 / (double)g3;
                        if (cost < best_cost - 1e-12) { best_cost = cost; best = {K, g0, g1, g2, g3}; }
                    }
    }
    if (env_n >= 2) best.G0 = std::max<long long>(1, env_g[0]);
    if (env_n >= 3) best.G1 = std::max<long long>(1, env_g[1]);
    if (env_n >= 4) best.G2 = std::max<long long>(1, env_g[2]);
    if (env_n >= 5) best.G3 = std::max<long long>(1, env_g[3]);
    if (best.K < 2) best.G0 = 1;
    if (best.K < 3) best.G1 = 1;
    if (best.K < 4) best.G2 = 1;
    if (best.K < 5) best.G3 = 1;
    return best;
}

template <int D, bool SPLIT, bool GT, int K>
ddks_status launch_kd(ddks_ctx* ctx, const CountPlan& pl, const ddks::CountArgs& a, cudaStream_t st) {
    return launch_count_t<D, SPLIT, GT, K>(ctx, pl, a, st);
}

template <int D, bool SPLIT>
ddks_status run_count_kd_t(ddks_ctx* ctx, const float* packed, int64_t n_P, int64_t n_Q, int shard_world,
                           int shard_rank, uint64_t* item_num, uint64_t* per_origin, cudaStream_t st,
                           unsigned long long* hist_out, unsigned long long* best_key) {
    using G = ddks::Geo<D, SPLIT>;
    const int64_t N = n_P + n_Q;
    const int DP = pad_dim(D);
    const bool gt = (ctx->flags & DDKS_FLAG_TIES_GT) != 0;
    const int64_t A = lcm_i64(G::ORIGINS, G::TILE);
    const int forced = (int)((ctx->flags >> DDKS_FLAG_KD_SHIFT) & 7u);
    // the tie-convention test variant (GT) is instantiated with one level only
    // mid N (< 80000 rows, one rank): bucket counting sorts (3 launches per level) instead of the exact radix sort
    // (~17 launches per level, latency-bound below ~10^5 rows). The bucket scatter places equal-bucket rows in
    // arbitrary (atomic) order, so the order is not reproducible from call to call: counts and results are exact
    // either way, but origin shards are defined on the order, so sharded runs (world > 1 and the shard rehearsal)
    // keep the deterministic radix sort. Each level costs ~35 us here, so at most 2 levels (C3: K = 2 1.20 ms vs
    // K = 3 1.47 ms per call). DDKS_KD_RADIX (test only) forces the radix sort.
    const bool bucket = N < 80000 && shard_world <= 1 && !getenv("DDKS_KD_RADIX");
    const KdChoice kc = kd_choose(D, std::min(n_P, n_Q), G::ORIGINS, 32 * G::R, G::TILE, A, gt ? 1 : forced,
                                  gt ? 1 : (bucket && !forced ? 2 : 5));
    const int K = kc.K;
    const int ib = std::max(1, bits_for((uint64_t)(N - 1)));
    const int tiles_rs = (int)((N + ddks::RS_TILE - 1) / ddks::RS_TILE);
    const int64_t n_tiles = (N + G::TILE - 1) / G::TILE;
    ddks_status s;
    if ((s = ensure(ctx, ctx->x0_keys0, (size_t)N * 8))) return s;
    if ((s = ensure(ctx, ctx->x0_keys1, (size_t)N * 8))) return s;
    if ((s = ensure(ctx, ctx->x0_hist, (size_t)tiles_rs * 256 * 4))) return s;
    if ((s = ensure(ctx, ctx->x0_pts, (size_t)(N + 4) * DP * 4))) return s;
    if ((s = ensure(ctx, ctx->x0_perm, (size_t)N * 4))) return s;
    if ((s = ensure(ctx, ctx->x0_boxes, (size_t)n_tiles * K * 2 * 4))) return s;
    if (K > 1) {
        if ((s = ensure(ctx, ctx->x0_pts2, (size_t)N * DP * 4))) return s;
        if ((s = ensure(ctx, ctx->x0_perm2, (size_t)N * 4))) return s;
    }
    uint64_t* k0 = (uint64_t*)ctx->x0_keys0.p;
    uint64_t* k1 = (uint64_t*)ctx->x0_keys1.p;
    uint32_t* hist = (uint32_t*)ctx->x0_hist.p;
    const int g = (int)std::max<int64_t>(1, std::min<int64_t>((N + 255) / 256, 148 * 16));
    const float* src_pts = packed;
    const int32_t* src_perm = nullptr;
    // mid-N ordering, preferred form: one thread-block cluster per label run (runs <= 65536 rows, <= 16384 cells)
    bool cluster_path = false;
    if (bucket && !getenv("DDKS_KD_FUSED")) {
        int64_t cmax = 1;
        const int64_t gl[4] = {kc.G0, kc.G1, kc.G2, kc.G3};
        for (int l = 0; l + 1 < K; ++l) cmax *= gl[l];
        cluster_path = K <= 4 && cmax < ddks::KDC_HW &&  // cells + 1 cell starts fit the offset words
                       std::max(n_P, n_Q) <= (int64_t)ddks::KDC_CS * ddks::KDC_T * ddks::KDC_RPT;
    }
    if (cluster_path) {
        if (K > 1) {
            if ((s = ensure(ctx, ctx->x0_pts2, (size_t)N * DP * 4))) return s;
            if ((s = ensure(ctx, ctx->x0_perm2, (size_t)N * 4))) return s;
        }
        static std::atomic<bool> attr_set[kMaxDevices] = {};
        if (!attr_set[ctx->device].load(std::memory_order_acquire)) {
            CU(cudaFuncSetAttribute(ddks::k_kdb_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, ddks::KDC_SMEM));
            attr_set[ctx->device].store(true, std::memory_order_release);
        }
        ddks::KdcArgs ca{};
        ca.pts = packed;
        ca.DP = DP;
        ca.K = K;
        ca.N = N;
        ca.n_P = n_P;
        ca.G0 = kc.G0;
        ca.G1 = kc.G1;
        ca.G2 = kc.G2;
        ca.A = A;
        ca.out[0] = (float*)ctx->x0_pts.p;
        ca.out[1] = (float*)ctx->x0_pts2.p;
        ca.perm[0] = (int32_t*)ctx->x0_perm.p;
        ca.perm[1] = (int32_t*)ctx->x0_perm2.p;
        ddks::k_kdb_cluster<<<2 * ddks::KDC_CS, ddks::KDC_T, ddks::KDC_SMEM, st>>>(ca);
        CHECK_LAUNCH();
        ctx->launches++;
    }
    if (bucket && !cluster_path) {
        // the whole ordering (ranges, K bucket-sort levels, pad rows, tile boxes) in one cooperative launch; its
        // histograms and ranges live in a buffer zeroed when allocated and left zeroed / reset by every launch
        int64_t hwords = 0, cells = 1;
        const int64_t gl[4] = {kc.G0, kc.G1, kc.G2, kc.G3};
        for (int l = 0; l < K; ++l) hwords += 2 * cells * ddks::KB_NBK, cells *= gl[l];
        int nsm = 148;
        CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device));
        nsm = std::min(nsm, ddks::KDF_MAXB);
        // layout: ranges [2][4][2] words, chunk totals [KDF_MAXB], histograms [hwords]
        const size_t kb_bytes = (size_t)(16 + ddks::KDF_MAXB + hwords) * 4;
        if (ctx->kdf_buf.bytes < kb_bytes) {
            if ((s = ensure(ctx, ctx->kdf_buf, kb_bytes))) return s;
            CU(cudaMemsetAsync(ctx->kdf_buf.p, 0, ctx->kdf_buf.bytes, st));
            ddks::k_kdb_range_init<<<1, 32, 0, st>>>((unsigned int*)ctx->kdf_buf.p, 8);  // ranges start at (~0, 0)
            CHECK_LAUNCH();
            ctx->launches++;
        }
        if ((s = ensure_zeroed(ctx, ctx->kdf_bar, 64, st))) return s;  // barrier: arrived stays 0 between launches
        if (K > 1) {
            if ((s = ensure(ctx, ctx->x0_pts2, (size_t)N * DP * 4))) return s;
            if ((s = ensure(ctx, ctx->x0_perm2, (size_t)N * 4))) return s;
        }
        ddks::KdbFusedArgs fa{};
        fa.pts = packed;
        fa.DP = DP;
        fa.K = K;
        fa.N = N;
        fa.n_P = n_P;
        fa.G0 = kc.G0;
        fa.G1 = kc.G1;
        fa.G2 = kc.G2;
        fa.A = A;
        fa.out[0] = (float*)ctx->x0_pts.p;
        fa.out[1] = (float*)ctx->x0_pts2.p;
        fa.perm[0] = (int32_t*)ctx->x0_perm.p;
        fa.perm[1] = (int32_t*)ctx->x0_perm2.p;
        fa.keys = (uint32_t*)k0;
        fa.rng = (uint32_t*)ctx->kdf_buf.p;
        fa.tot = fa.rng + 16;
        fa.hist = fa.tot + ddks::KDF_MAXB;
        fa.bar = (uint32_t*)ctx->kdf_bar.p;
        fa.boxes = (float*)ctx->x0_boxes.p;
        fa.TILE = G::TILE;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)nsm, 1, 1);
        cfg.blockDim = dim3(ddks::KDF_T, 1, 1);
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;  // every CTA resident: the grid barriers cannot deadlock
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CU(cudaLaunchKernelEx(&cfg, ddks::k_kdb_fused, fa));
        ctx->launches++;
    }
    for (int level = 0; level < (bucket ? 0 : K); ++level) {
        const int64_t gl[4] = {kc.G0, kc.G1, kc.G2, kc.G3};
        int64_t cells = 1;
        for (int l = 0; l < level; ++l) cells *= gl[l];
        const int cb = cells > 1 ? bits_for((uint64_t)(cells - 1)) : 0;
        // the full 32-bit order key whenever it fits (truncated keys tie points across cut points, and the touching
        // cell ranges then leave bits open: C5 709 -> 733 ms with 16 / 24-bit keys); only the top 1 + cb + kb bits
        // are sorted, so the index bits below them cost no radix passes
        const int kb = std::min(32, 63 - cb - ib);
        const int passes = (1 + cb + kb + 7) / 8;
        const int shift_begin = std::max(0, 64 - 8 * passes);
        ddks::k_kd_keys<<<g, 256, 0, st>>>(src_pts, DP, N, n_P, level, kc.G0, kc.G1, kc.G2, kc.G3, A, ib, cb, kb, k0);
        CHECK_LAUNCH();
        ctx->launches++;
        uint64_t* sorted = nullptr;
        if ((s = radix_sort_keys(ctx, k0, k1, N, 1, shift_begin, hist, st, &sorted))) return s;
        // the last level lands in x0_pts / x0_perm; earlier ones alternate with x0_pts2 / x0_perm2
        const bool fin = ((K - 1 - level) % 2) == 0;
        float* dst_pts = (float*)(fin ? ctx->x0_pts.p : ctx->x0_pts2.p);
        int32_t* dst_perm = (int32_t*)(fin ? ctx->x0_perm.p : ctx->x0_perm2.p);
        ddks::k_permute_rows<<<g, 256, 0, st>>>(src_pts, DP, N, sorted, ib, src_perm, dst_pts, dst_perm);
        CHECK_LAUNCH();
        ctx->launches++;
        src_pts = dst_pts;
        src_perm = dst_perm;
    }
    bool boxes_done = bucket && !cluster_path;  // the fused mid-N ordering wrote the pad rows and the tile boxes
    // TEST ONLY (DDKS_KD_SHUFFLE=m): scramble the rows inside each label run (position p -> p * m mod n, m odd and
    // coprime to n) after the kd sort. The counts must not depend on the order -- only the speed does.
    if (const char* e = getenv("DDKS_KD_SHUFFLE")) {
        const long long m = atoll(e);
        if (m > 1) {
            if ((s = ensure(ctx, ctx->x0_pts2, (size_t)N * DP * 4))) return s;
            if ((s = ensure(ctx, ctx->x0_perm2, (size_t)N * 4))) return s;
            CU(cudaMemcpyAsync(ctx->x0_pts2.p, ctx->x0_pts.p, (size_t)N * DP * 4, cudaMemcpyDeviceToDevice, st));
            CU(cudaMemcpyAsync(ctx->x0_perm2.p, ctx->x0_perm.p, (size_t)N * 4, cudaMemcpyDeviceToDevice, st));
            boxes_done = false;  // the boxes must describe the shuffled rows
            ddks::k_shuffle_runs<<<g, 256, 0, st>>>((const float*)ctx->x0_pts2.p, (const int32_t*)ctx->x0_perm2.p, DP,
                                                     N, n_P, m, (float*)ctx->x0_pts.p, (int32_t*)ctx->x0_perm.p);
            CHECK_LAUNCH();
            ctx->launches++;
        }
    }
    float* spts = (float*)ctx->x0_pts.p;
    if (!boxes_done) {
        CU(cudaMemsetAsync(spts + N * DP, 0, 4 * DP * 4, st));  // the prefetch past the last row reads zeros
        ddks::k_tile_boxes<<<(int)std::max<int64_t>(1, std::min<int64_t>((n_tiles + 7) / 8, 148 * 16)), 256, 0, st>>>(
            spts, DP, N, G::TILE, K, (float*)ctx->x0_boxes.p);
        CHECK_LAUNCH();
        ctx->launches++;
    }
    const uint64_t gg = gcd_u64((uint64_t)n_P, (uint64_t)n_Q);
    const uint32_t a_ = (uint32_t)((uint64_t)n_Q / gg), b_ = (uint32_t)((uint64_t)n_P / gg);
    // all N origins (positions of the kd order); shard r of W takes origin blocks r, r + W, r + 2W, ... so every
    // rank gets the same mix of cells (contiguous shards differ by ~10 % in decided bits at C5)
    CountPlan pl{1, (int32_t)N, (int32_t)n_P, 0, (int32_t)N, n_P, n_Q, SPLIT,
                 SPLIT ? 32767 : (int64_t)(32767 / std::max(a_, b_)), shard_world, shard_rank};
    ddks::CountArgs a{};
    a.pts = spts;
    a.item_stride = N * DP;
    a.N = (int32_t)N;
    a.n_P = (int32_t)n_P;
    a.o_begin = 0;
    a.o_end = (int32_t)N;
    a.incP = SPLIT ? 1u : a_;
    a.incQ = SPLIT ? 1u : 0u - b_;
    a.gg = gg;
    a.aQ = (int64_t)a_;
    a.bP = (int64_t)b_;
    a.item_num = item_num;
    a.per_origin = per_origin;
    a.perm = (const int32_t*)ctx->x0_perm.p;
    a.boxes = (const float*)ctx->x0_boxes.p;
    a.hist = SPLIT ? hist_out : nullptr;
    a.hist_stride = n_Q + 1;
    a.best_key = best_key;
    ctx->kd_levels = K;
    ctx->rank_lanes = 0;
    if (gt) return launch_kd<D, SPLIT, true, 1>(ctx, pl, a, st);
    if (K == 1) return launch_kd<D, SPLIT, false, 1>(ctx, pl, a, st);
    if constexpr (D >= 2) {
        if (K == 2) return launch_kd<D, SPLIT, false, 2>(ctx, pl, a, st);
    }
    if constexpr (D >= 3) {
        if (K == 3) return launch_kd<D, SPLIT, false, 3>(ctx, pl, a, st);
    }
    if constexpr (D >= 4 && DDKS_KD_MAX >= 4) {
        if (K == 4) return launch_kd<D, SPLIT, false, 4>(ctx, pl, a, st);
    }
    if constexpr (D >= 5 && DDKS_KD_MAX >= 5) {
        if (K == 5) return launch_kd<D, SPLIT, false, 5>(ctx, pl, a, st);
    }
    return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "kd levels %d for d=%d", K, D);
}

template <int D>
ddks_status run_count_kd_d(ddks_ctx* ctx, const float* packed, int64_t n_P, int64_t n_Q, int shard_world,
                           int shard_rank, uint64_t* item_num, uint64_t* per_origin, cudaStream_t st, bool split,
                           unsigned long long* hist, unsigned long long* best_key) {
    return split ? run_count_kd_t<D, true>(ctx, packed, n_P, n_Q, shard_world, shard_rank, item_num, per_origin, st, hist,
                                           best_key)
                 : run_count_kd_t<D, false>(ctx, packed, n_P, n_Q, shard_world, shard_rank, item_num, per_origin, st, hist,
                                            best_key);
}

}  // namespace ddks_host
