// ddks_launch.cuh — host-side launch of the count kernel (segment planning, accumulators, finaliser), shared by the
// translation units that instantiate k_count (ddks_api.cu: position order; ddks_api_kd*.cu: kd order).
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <utility>

#include "ddks_kernels.cuh"
#include "ddks_internal.h"

namespace ddks_host {

struct CountPlan {
    int64_t B;
    int32_t N, n_P, o_begin, o_end;
    int64_t nP, nQ;
    bool split;      // SPLIT counters (c_P, c_Q separately)
    int64_t window;  // max points per segment so no 16-bit counter half leaves int16
    int32_t blk_stride = 1, blk_off = 0;  // this launch takes origin blocks blk_off, blk_off + blk_stride, ...
};

template <int D, bool SPLIT, bool GT, int KX = 0, bool WX = false, bool SMALL = false>
ddks_status launch_count_t(ddks_ctx* ctx, const CountPlan& pl, ddks::CountArgs a, cudaStream_t st) {
    using G = ddks::Geo<D, SPLIT, SMALL>;
    auto kern = ddks::k_count<D, SPLIT, GT, KX, WX, SMALL>;
    // function attributes are per device: remember which devices this instantiation was configured on (atomics:
    // contexts on different host threads may launch the same instantiation; setting the attribute twice is harmless)
    static std::atomic<bool> attr_done[kMaxDevices] = {};
    if (ctx->device >= kMaxDevices) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "device index %d >= %d", ctx->device, kMaxDevices);
    if (!attr_done[ctx->device].load(std::memory_order_acquire)) {
        CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM_BYTES));
        attr_done[ctx->device].store(true, std::memory_order_release);
    }
    const int n_orig = pl.o_end - pl.o_begin;
    const int blocks_all = (n_orig + G::ORIGINS - 1) / G::ORIGINS;
    const int blocks_o = blocks_all > pl.blk_off ? (blocks_all - pl.blk_off + pl.blk_stride - 1) / pl.blk_stride : 0;
    if (blocks_o == 0) return DDKS_OK;  // no origin block falls to this shard
    a.warp_major = (KX > 0 || WX) ? 1 : 0;  // must match k_count's origin_of
    a.blk_stride = pl.blk_stride;
    a.blk_off = pl.blk_off;
    // accumulator slots per item: the origin offsets themselves when slots and origins coincide (plain mapping, all
    // blocks), else whole blocks of slots (strided shards; warp-major slots of kd / WX counts)
    a.acc_stride = (pl.blk_stride == 1 && !a.warp_major) ? n_orig : blocks_o * G::ORIGINS;
    const int n_tiles = (pl.N + G::TILE - 1) / G::TILE;
    // segment length: at most the int16 flush window. Among the segment counts that respect it, pick the one with
    // the least modelled time: waves x per-CTA cost, where a CTA costs its segment's points (x its origins) plus the
    // flush of NB int32 partials per origin (global atomics; ~FLUSH_COST point-equivalents each) and the setup.
    static std::atomic<int> per_sm_dev[kMaxDevices] = {};
    int per_sm = per_sm_dev[ctx->device].load(std::memory_order_relaxed);
    if (!per_sm) {
        CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, G::T, G::SMEM_BYTES));
        per_sm = std::max(per_sm, 1);
        per_sm_dev[ctx->device].store(per_sm, std::memory_order_relaxed);
    }
    int nsm = 148;
    CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device));
    const int64_t slots = (int64_t)nsm * per_sm;
    const int w_tiles = std::max(1, (int)(pl.window / G::TILE));
    const int min_segs = (n_tiles + w_tiles - 1) / w_tiles;
    const int64_t base_ctas = pl.B * blocks_o;
    int segs = min_segs;
    if (WX && min_segs > 1) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "warp-level x0 count needs one point segment");
    if (!WX && !(ctx->flags & DDKS_FLAG_FORCE_DIRECT)) {
        constexpr double FLUSH_COST = 2.0, SETUP_COST = 2.0 * G::TILE;  // calibrated on C3 (segs 2..16 sweep)
        // segments need the partials' memset and the k_finalize launch (~5 us): worth ~4 tiles of one CTA's work
        constexpr double FIN_COST = 4.0 * G::TILE;
        double best = 1e300;
        const int max_segs = (int)std::min<int64_t>(n_tiles, std::max<int64_t>(min_segs, (16 * slots + base_ctas - 1) / base_ctas));
        for (int sg = min_segs; sg <= max_segs; ++sg) {
            const int tps = (n_tiles + sg - 1) / sg;
            const int real = (n_tiles + tps - 1) / tps;
            if (real != sg) continue;
            const int64_t ctas = base_ctas * sg;
            const int64_t waves = (ctas + slots - 1) / slots;
            const double cta = (double)tps * G::TILE + SETUP_COST + (sg > 1 ? FLUSH_COST * G::NB : 0.0);
            const double cost = (double)waves * cta + (sg > 1 ? FIN_COST : 0.0);
            if (cost < best * (1.0 - 1e-9)) { best = cost; segs = sg; }
        }
        if (const char* e = getenv("DDKS_SEGS")) segs = std::max(min_segs, std::min(n_tiles, atoi(e)));  // tuning override
    }
    const int tiles_per_seg = (n_tiles + segs - 1) / segs;
    segs = (n_tiles + tiles_per_seg - 1) / tiles_per_seg;
    a.seg_points = tiles_per_seg * G::TILE;
    if (segs > 0x7fffffff / 2) return fail(ctx, DDKS_ERR_TOO_LARGE, "too many point segments");
    if (segs > 1) {
        // int32 partials, zeroed per launch (measured: re-zeroing them in k_finalize instead cost C3 +160 us: the
        // finaliser's zero stores serialise its loads; one memset kernel is ~10 us)
        const size_t acc_bytes = (size_t)pl.B * G::NB * (size_t)a.acc_stride * 4;
        ddks_status s = ensure(ctx, ctx->accum, acc_bytes);
        if (s) return s;
        CU(cudaMemsetAsync(ctx->accum.p, 0, acc_bytes, st));
        a.accum = (int32_t*)ctx->accum.p;
    } else {
        a.accum = nullptr;
    }
    if (pl.B > 65535) return fail(ctx, DDKS_ERR_TOO_LARGE, "grid too large");
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
        ddks_status s = ensure_prof(ctx);
        if (s) return s;
        a.clk = (unsigned long long*)ctx->prof_clk.p;
    }
    // grid: x = point segment, y = origin block (chunks of 65535; DDKS_GRIDY, TEST ONLY, lowers the chunk), z = item
    int ych = 65535;
    if (const char* e = getenv("DDKS_GRIDY")) ych = std::max(1, std::min(65535, atoi(e)));
    for (int y0 = 0; y0 < blocks_o; y0 += ych) {
        a.blk_base = y0;
        dim3 grid((unsigned)segs, (unsigned)std::min(ych, blocks_o - y0), (unsigned)pl.B);
        kern<<<grid, G::T, G::SMEM_BYTES, st>>>(a);
        CHECK_LAUNCH();
        ctx->launches++;
    }
    if (ev.first) {
        CU(record_event(ev.second, st));
        ctx->ev_pending.push_back(ev);
        ctx->ev_recycle.push_back(1);
        // origins of this launch: its blocks, less the missing tail of the last block when that block is its own
        const bool last_own = (blocks_all - 1 - pl.blk_off) % pl.blk_stride == 0;
        const uint64_t own = (uint64_t)blocks_o * G::ORIGINS - (last_own ? (uint64_t)blocks_all * G::ORIGINS - n_orig : 0);
        ctx->ev_pairs.push_back((uint64_t)pl.B * own * (uint64_t)pl.N);
    }
    if (segs > 1) {
        const int64_t total = pl.B * a.acc_stride;
        const int threads = 256;
        constexpr int NQ = 1 << D, TPS = NQ >= 256 ? 8 : (NQ >= 128 ? 4 : (NQ >= 64 ? 2 : 1));
        const int64_t per_cta = threads / TPS;  // slots per CTA iteration (k_finalize)
        const int blocks = (int)std::min<int64_t>((total + per_cta - 1) / per_cta, 148 * 16);
        ddks::k_finalize<D, SPLIT, SMALL><<<blocks, threads, 0, st>>>(a, pl.B);
        CHECK_LAUNCH();
        ctx->launches++;
    }
    return DDKS_OK;
}

}  // namespace ddks_host
