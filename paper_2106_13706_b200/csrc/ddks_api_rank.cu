// ddks_api_rank.cu — host launch of the rank-lane count (ddks_rank.cuh): position-ordered single statistics at
// d = 2..8 with the >= convention; DIFF counters in one launch, SPLIT counters (c_P and c_Q apart) in two launches
// over the P rows and the Q rows. The finaliser is the one of launch_count_t (ddks_launch.cuh); the partial counters
// use the same [bin][origin offset] layout, so k_finalize<D, SPLIT> reads them unchanged.
#include "ddks_launch.cuh"
#include "ddks_rank.cuh"

namespace ddks_host {
namespace {

template <int D>
ddks_status launch_count_rank_d(ddks_ctx* ctx, const CountPlan& pl, ddks::CountArgs a, cudaStream_t st) {
    using G = ddks::RankGeo<D>;
    auto kern = ddks::k_count_rank<D, DDKS_RK_R>;
    constexpr int TPB = G::ORIGINS / DDKS_RK_R;
    constexpr int NQ = 1 << D;
    if (pl.B != 1 || pl.blk_stride != 1 || pl.blk_off != 0)
        return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "rank-lane count: one statistic over a contiguous shard");
    static std::atomic<bool> attr_done[kMaxDevices] = {};
    if (ctx->device >= kMaxDevices) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "device index %d >= %d", ctx->device, kMaxDevices);
    if (!attr_done[ctx->device].load(std::memory_order_acquire)) {
        CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM_BYTES));
        attr_done[ctx->device].store(true, std::memory_order_release);
    }
    const int n_orig = pl.o_end - pl.o_begin;
    const int blocks_o = (n_orig + G::ORIGINS - 1) / G::ORIGINS;
    if (blocks_o == 0) return DDKS_OK;
    a.warp_major = 0;
    a.blk_stride = 1;
    a.blk_off = 0;
    a.acc_stride = n_orig;
    a.perm = nullptr;
    a.boxes = nullptr;
    static std::atomic<int> per_sm_dev[kMaxDevices] = {};
    int per_sm = per_sm_dev[ctx->device].load(std::memory_order_relaxed);
    if (!per_sm) {
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, TPB, G::SMEM_BYTES));
        per_sm = std::max(per_sm, 1);
        per_sm_dev[ctx->device].store(per_sm, std::memory_order_relaxed);
    }
    int nsm = 148;
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device));
    const int64_t slots = (int64_t)nsm * per_sm;
    // SPLIT counters (c_P and c_Q kept apart: the significance's M_T histogram, or sample sizes whose DIFF counters
    // would overflow): the same kernel counts the P rows into bins [0, 2^d) and, in a second launch, the Q rows into
    // bins [2^d, 2^(d+1)) of the accumulator, every pair adding +1 -- together the N^2 pairs of one DIFF launch; the
    // SPLIT finaliser forms |c_P a - c_Q b| and histograms c_Q. Always stream-K (the finaliser reads the partials).
    const int n_pass = pl.split ? 2 : 1;
    const int32_t rng[2][2] = {{0, pl.split ? (int32_t)pl.nP : pl.N}, {(int32_t)pl.nP, pl.N}};
    // flush window in tiles. DIFF: a chunk's final counter c_P a - c_Q b lies in [-#Q b, #P a] (P rows precede Q rows),
    // so when n_P a and n_Q b both fit int16 any chunk does (C3: the whole point set); else the generic window.
    // SPLIT: a counter grows by one per point, so 32767 points fit
    const int64_t ga = (int64_t)pl.nQ / (int64_t)gcd_u64((uint64_t)pl.nP, (uint64_t)pl.nQ);
    const int64_t gb = (int64_t)pl.nP / (int64_t)gcd_u64((uint64_t)pl.nP, (uint64_t)pl.nQ);
    const bool whole = !pl.split && pl.nP * ga <= 32767 && pl.nQ * gb <= 32767;
    const int n_tiles_all = (pl.N + G::TILE - 1) / G::TILE;
    const int chunk_all = whole ? n_tiles_all : std::max(1, (int)(pl.window / G::TILE));
    // direct (one CTA per whole block, in-kernel finalisation) when the blocks fill the SMs in one wave and fit a
    // window; else stream-K over (block, tile) units with one persistent CTA per slot (every SM the same number of
    // tiles; a CTA flushes the partials of the <= 2-3 blocks it visits, k_finalize sums them). Modelled in tiles:
    // direct = waves x n_tiles; stream-K = units / slots + ~3 tiles of flush per CTA + ~4 tiles for the memset +
    // k_finalize.
    const int64_t units_all = (int64_t)blocks_o * n_tiles_all;
    const double cost_direct = chunk_all >= n_tiles_all ? (double)((blocks_o + slots - 1) / slots) * n_tiles_all : 1e300;
    const double cost_sk = (double)((units_all + slots - 1) / slots) + 3.0 + 4.0;
    bool direct = !pl.split && (cost_direct <= cost_sk || (ctx->flags & DDKS_FLAG_FORCE_DIRECT));
    if (direct && chunk_all < n_tiles_all) direct = false;  // FORCE_DIRECT cannot hold a point set beyond the window
    if (const char* e = getenv("DDKS_RANK_SK")) direct = !pl.split && atoi(e) == 0 && chunk_all >= n_tiles_all;  // tuning override
    a.seg_points = n_tiles_all * G::TILE;
    if (!direct) {
        const size_t acc_bytes = (size_t)n_pass * NQ * (size_t)a.acc_stride * 4;
        ddks_status s = ensure(ctx, ctx->accum, acc_bytes);
        if (s) return s;
        CU(cudaMemsetAsync(ctx->accum.p, 0, acc_bytes, st));
        a.accum = (int32_t*)ctx->accum.p;
    } else {
        a.accum = nullptr;
    }
    // V_k of every origin block (Eytzinger order)
    ddks_status s = ensure(ctx, ctx->rank_v, (size_t)blocks_o * D * G::VW * 4);
    if (s) return s;
    float* vs = (float*)ctx->rank_v.p;
    for (int y0 = 0; y0 < blocks_o; y0 += 65535) {
        // grid.x = block, y = dim; the block index is offset through o_begin
        const int nb = std::min(65535, blocks_o - y0);
        ddks::k_rank_sort<D><<<dim3((unsigned)nb, D), 256, 0, st>>>(a.pts, ddks::padded_dim<D>(),
                                                                   a.o_begin + y0 * G::ORIGINS, a.o_end,
                                                                   vs + (size_t)y0 * D * G::VW);
        CHECK_LAUNCH();
        ctx->launches++;
    }
    std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
    if (ctx->flags & DDKS_FLAG_PROFILE) {
        if (!ctx->ev_free.empty()) {
            ev = ctx->ev_free.back();
            ctx->ev_free.pop_back();
        } else {
            CU(cudaEventCreate(&ev.first));
            CU(cudaEventCreate(&ev.second));
        }
        CU(record_event(ev.first, st));
        ddks_status s2 = ensure_prof(ctx);
        if (s2) return s2;
        a.clk = (unsigned long long*)ctx->prof_clk.p;
    }
    int32_t* const acc0 = a.accum;
    const int32_t N_all = a.N, nP_all = a.n_P;
    for (int ps = 0; ps < n_pass; ++ps) {
        const int32_t rows = rng[ps][1] - rng[ps][0];
        if (rows <= 0) continue;
        ddks::RankArgs ra{};
        ra.vsorted = vs;
        ra.pt_rows = a.pts + (size_t)rng[ps][0] * ddks::padded_dim<D>();
        a.N = rows;                                          // rows of this launch ...
        a.n_P = pl.split ? (ps == 0 ? rows : 0) : nP_all;    // ... of which the first n_P add inc P
        ra.n_tiles = (rows + G::TILE - 1) / G::TILE;
        ra.chunk_tiles = whole ? ra.n_tiles : std::max(1, (int)(pl.window / G::TILE));
        ra.units = (int64_t)blocks_o * ra.n_tiles;
        const int64_t grid = direct ? blocks_o : std::min<int64_t>(slots, ra.units);
        if (grid > 0x7fffffff) return fail(ctx, DDKS_ERR_TOO_LARGE, "rank-lane count: too many origin blocks");
        a.accum = acc0 ? acc0 + (size_t)ps * NQ * (size_t)a.acc_stride : nullptr;
        kern<<<(unsigned)grid, TPB, G::SMEM_BYTES, st>>>(a, ra);
        CHECK_LAUNCH();
        ctx->launches++;
    }
    a.N = N_all;
    a.n_P = nP_all;
    a.accum = acc0;
    if (ev.first) {
        CU(record_event(ev.second, st));
        ctx->ev_pending.push_back(ev);
        ctx->ev_recycle.push_back(1);
        ctx->ev_pairs.push_back((uint64_t)n_orig * (uint64_t)pl.N);
    }
    if (!direct) {
        const int64_t total = a.acc_stride;
        const int threads = 256;
        constexpr int TPS = NQ >= 256 ? 8 : (NQ >= 128 ? 4 : (NQ >= 64 ? 2 : 1));
        const int64_t per_cta = threads / TPS;
        const int blocks = (int)std::min<int64_t>((total + per_cta - 1) / per_cta, 148 * 16);
#ifndef DDKS_RANK_NO_SPLIT_FIN
        if (pl.split) ddks::k_finalize<D, true, false><<<blocks, threads, 0, st>>>(a, 1);
        else
#endif
            ddks::k_finalize<D, false, false><<<blocks, threads, 0, st>>>(a, 1);
        CHECK_LAUNCH();
        ctx->launches++;
    }
    return DDKS_OK;
}

}  // namespace

ddks_status run_count_rank(ddks_ctx* ctx, const float* packed, int d, int64_t n_P, int64_t n_Q, int64_t o_begin,
                           int64_t o_end, uint64_t* item_num, uint64_t* per_origin, cudaStream_t st,
                           unsigned long long* best_key, bool split, unsigned long long* hist) {
    const int64_t N = n_P + n_Q;
    const uint64_t g = gcd_u64((uint64_t)n_P, (uint64_t)n_Q);
    const uint64_t a_ = (uint64_t)n_Q / g, b_ = (uint64_t)n_P / g;
    // DIFF counters (the caller checked diff_counters_ok): a 16-bit half stays in int16 over 32767 / max(a, b) points;
    // SPLIT counters grow by one per point
    const int64_t window = split ? 32767 : (int64_t)(32767 / std::max(a_, b_));
    CountPlan pl{1, (int32_t)N, (int32_t)n_P, (int32_t)o_begin, (int32_t)o_end, n_P, n_Q, split, window};
    ddks::CountArgs a{};
    a.pts = packed;
    a.item_stride = N * pad_dim(d);
    a.N = (int32_t)N;
    a.n_P = (int32_t)n_P;
    a.o_begin = (int32_t)o_begin;
    a.o_end = (int32_t)o_end;
    a.incP = split ? 1u : (uint32_t)a_;
    a.incQ = split ? 1u : (uint32_t)(0u - (uint32_t)b_);
    a.gg = g;
    a.aQ = (int64_t)a_;
    a.bP = (int64_t)b_;
    a.item_num = item_num;
    a.per_origin = per_origin;
    a.hist = split ? hist : nullptr;
    a.hist_stride = n_Q + 1;
    a.best_key = best_key;
    ctx->rank_lanes = 1;
    switch (d) {
        case 2: return launch_count_rank_d<2>(ctx, pl, a, st);
        case 3: return launch_count_rank_d<3>(ctx, pl, a, st);
        case 4: return launch_count_rank_d<4>(ctx, pl, a, st);
        case 5: return launch_count_rank_d<5>(ctx, pl, a, st);
        case 6: return launch_count_rank_d<6>(ctx, pl, a, st);
        case 7: return launch_count_rank_d<7>(ctx, pl, a, st);
        case 8: return launch_count_rank_d<8>(ctx, pl, a, st);
    }
    return fail(ctx, DDKS_ERR_DIM_UNSUPPORTED, "rank-lane count: d=%d", d);
}

}  // namespace ddks_host
