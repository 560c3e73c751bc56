// ddks_api.cu — host side of libddks.so: the C ABI declared in include/ddks.h.
//
// Context = device + grow-only workspace + (world > 1, or the NCCL_SELF test flag) an NCCL communicator (NCCL 2.28.9, the
// copy torch bundles). A statistic: argument checks -> optional H2D of host inputs -> k_pack (validate + pack) ->
// [kd ordering] -> k_count (classify + count + per-origin max + packed argmax key) [-> k_finalize] -> (world > 1) one
// all-gather of the per-rank records -> one D2H -> sync -> host combine; N <= 8192 on one rank: the single fused
// k_count_small launch instead (ddks_small.cuh). Repeated identical ddks_stat calls replay a captured CUDA graph.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <type_traits>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ddks_kernels.cuh"
#include "ddks_radix.cuh"
#include "ddks_small.cuh"
#include "ddks_perm_mma.cuh"
#include "ddks_internal.h"
#include "ddks_launch.cuh"

#define DDKS_VERSION "0.1.0-sm100a"

thread_local std::string g_create_err;

namespace ddks_host {

ddks_status fail(ddks_ctx* c, ddks_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    else g_create_err = buf;
    return s;
}

ddks_status ensure(ddks_ctx* ctx, DevBuf& b, size_t bytes) {
    if (bytes <= b.bytes) return DDKS_OK;
    if (b.p) cudaFree(b.p);
    // a new allocation may reuse the old address: the self-cleaning count buffers lose their known-zero state
    if (&b == &ctx->vox_cnt) ctx->vox_zero_p = nullptr;
    if (&b == &ctx->rdb_cnt) ctx->rdb_zero_p = nullptr;
    b.p = nullptr;
    b.bytes = 0;
    size_t want = std::max(bytes, (size_t)256);
    ctx->alloc_epoch++;  // invalidates captured graphs (they hold the old pointers)
    cudaError_t e = cudaMalloc(&b.p, want);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, DDKS_ERR_OOM, "cudaMalloc(%zu) failed: %s", want, cudaGetErrorString(e));
    }
    b.bytes = want;
    return DDKS_OK;
}

ddks_status ensure_zeroed(ddks_ctx* ctx, DevBuf& b, size_t bytes, cudaStream_t st) {
    if (bytes <= b.bytes) return DDKS_OK;
    ddks_status s = ensure(ctx, b, bytes);
    if (s) return s;
    CU(cudaMemsetAsync(b.p, 0, b.bytes, st));
    return DDKS_OK;
}

ddks_status ensure_prof(ddks_ctx* ctx) {
    if (ctx->prof_clk.p) return DDKS_OK;
    ddks_status s = ensure(ctx, ctx->prof_clk, 32);
    if (s) return s;
    CU(cudaMemset(ctx->prof_clk.p, 0, 32));
    return DDKS_OK;
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Bring an input to the device: device pointers are used in place, host pointers are copied on `st`.
ddks_status stage_input(ddks_ctx* ctx, const void* src, size_t bytes, DevBuf& buf, cudaStream_t st, const void** out) {
    if (is_device_ptr(src)) {
        *out = src;
        return DDKS_OK;
    }
    ddks_status s = ensure(ctx, buf, bytes);
    if (s) return s;
    CU(cudaMemcpyAsync(buf.p, src, bytes, cudaMemcpyHostToDevice, st));
    *out = buf.p;
    return DDKS_OK;
}

uint64_t gcd_u64(uint64_t a, uint64_t b) {
    while (b) {
        uint64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

ddks_status check_sizes(ddks_ctx* ctx, int64_t n_P, int64_t n_Q, int32_t d) {
    if (n_P < 0 || n_Q < 0) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "negative sample size");
    if (n_P == 0 || n_Q == 0) return fail(ctx, DDKS_ERR_EMPTY_SAMPLE, "empty sample (n_P=%lld, n_Q=%lld)",
                                          (long long)n_P, (long long)n_Q);
    if (d < 1 || d > 8) return fail(ctx, DDKS_ERR_DIM_UNSUPPORTED, "d=%d not in [1, 8]", d);
    if (n_P + n_Q >= (int64_t(1) << 31)) return fail(ctx, DDKS_ERR_TOO_LARGE, "n_P + n_Q >= 2^31");
    const double den = (double)n_P * (double)n_Q;
    if (den >= 9007199254740992.0) return fail(ctx, DDKS_ERR_TOO_LARGE, "n_P * n_Q >= 2^53");
    return DDKS_OK;
}

int pad_dim(int d) { return d <= 4 ? 4 : 8; }

// ------------------------------------------------------------------------------------- count dispatch
// DIFF counters fit (|c_P a - c_Q b| stays in int32 and the int16 window is >= 4096 points); else SPLIT
bool diff_counters_ok(int64_t n_P, int64_t n_Q);

// the rank-lane count (ddks_rank.cuh) takes a position-ordered statistic at d = 3 and 5..8 in its measured range
// (d = 2..8 at any size with DDKS_FLAG_FORCE_RANK); the >= convention only; not for the small geometry. force_split:
// the caller needs SPLIT counters (significance); sample sizes whose DIFF counters would overflow need them too.
bool rank_applicable(ddks_ctx* ctx, int d, int64_t n_P, int64_t n_Q, bool force_split) {
    if (ctx->flags & (DDKS_FLAG_NO_RANK | DDKS_FLAG_TIES_GT)) return false;
    if (d < 2 || d > 8 || n_P + n_Q <= ddks::kSmallN) return false;
    const bool split = force_split || !diff_counters_ok(n_P, n_Q);
    if (ctx->flags & DDKS_FLAG_FORCE_RANK) return true;
    const int64_t N = n_P + n_Q;
    if (split) {
        // SPLIT (two launches, +1 per pair; ddks_api_rank.cu) against the FP32 SPLIT counts, kd-ordered where that
        // applies, which run 6 warps per SM at d = 8 (microbench/rank_split_ab.py, profiles/r2f_rank_split_ab.txt; warm
        // ms, significance | statistic with coprime sizes): d = 8 0.46 vs 1.20 | 0.33 vs 0.58 at N = 2e4, 1.14 vs 1.69 |
        // 0.93 vs 1.48 at 4e4 (C3), 20.6 vs 31.6 | 19.7 vs 30.4 at 2e5; d = 7 0.42 vs 0.49 at 2e4, 20.5 vs 22.4 | 19.6 vs
        // 21.0 at 2e5, slower at 1e4; d = 6 0.35 vs 0.40 at 2e4, 4.10 vs 4.98 | 3.57 vs 3.98 at 1e5, even at 2e5,
        // slower at 1e4; d = 5 0.85 vs 0.97 | 0.59 vs 0.71 at 4e4, 3.77 vs 4.04 | 3.17 vs 2.97 at 1e5; d = 3 never
        switch (d) {
            case 8: return N <= 600000;
            case 7: return N >= 15000 && N <= 250000;
            case 6: return N >= 15000 && N <= 150000;
            case 5: return N >= 30000 && N <= 90000;
        }
        return false;
    }
    // measured against the kd-ordered and position-ordered FP32 counts (microbench/rank_ab.py,
    // profiles/r2e_rank_ab.txt, r2f_rank_ab.txt; warm call times). d = 8 (three rank words): faster at N = 1e4 .. 4e5
    // (C3 0.88 vs 1.17 ms; 78 vs 82 ms at 4e5, the kd count's decided bits catch up beyond); d = 7: up to N ~ 5e4;
    // d = 6 (two words): 0.64 vs 0.89 ms at 4e4, 3.48 vs 3.87 at 1e5, 54 vs 46 at 4e5; d = 5: 0.58 vs 0.67 at 4e4,
    // 3.21 vs 3.10 at 1e5; d = 3 (one word; C2 0.156 vs 0.164 ms): 0.430 vs 0.453 at 4e4, 2.34 vs 2.01 at 1e5;
    // d = 4 ties and d = 2 loses (their FP32 counts are 9.6 / 5.7 instructions per pair already). Finer sweep
    // (N = 6e4, 8e4, 1.5e5, 2e5; call ms rank vs kd): d = 7 1.85 / 1.91, 3.23 / 3.09; d = 6 1.31 / 1.62, 2.26 / 2.70,
    // 7.71 / 8.13, 13.6 / 13.2; d = 5 1.20 / 1.23, 2.08 / 2.14, 7.08 / 6.11; d = 3 0.860 / 0.880, 1.477 / 1.467
    switch (d) {
        case 8: return N <= 600000;
        case 7: return N <= 70000;
        case 6: return N <= 170000;
        case 5: return N <= 90000;
        case 3: return N <= 65000;
    }
    return false;
}

template <int D>
ddks_status launch_count_d(ddks_ctx* ctx, const CountPlan& pl, const ddks::CountArgs& a, cudaStream_t st, bool wx) {
    const bool gt = (ctx->flags & DDKS_FLAG_TIES_GT) != 0;
    if constexpr (D >= 2) {
        // rows pre-sorted by x_0 inside every label run (k_pack_sorted) and one point segment: warp-level bit 0
        if (wx && !gt && pl.N <= pl.window)
            return pl.split ? launch_count_t<D, true, false, 0, true>(ctx, pl, a, st)
                            : launch_count_t<D, false, false, 0, true>(ctx, pl, a, st);
    }
    if (pl.B == 1 && pl.N <= ddks::kSmallN) {  // few points: the small geometry (more, smaller CTAs)
        if (pl.split) return gt ? launch_count_t<D, true, true, 0, false, true>(ctx, pl, a, st)
                                : launch_count_t<D, true, false, 0, false, true>(ctx, pl, a, st);
        return gt ? launch_count_t<D, false, true, 0, false, true>(ctx, pl, a, st)
                  : launch_count_t<D, false, false, 0, false, true>(ctx, pl, a, st);
    }
    if (pl.split) return gt ? launch_count_t<D, true, true>(ctx, pl, a, st) : launch_count_t<D, true, false>(ctx, pl, a, st);
    return gt ? launch_count_t<D, false, true>(ctx, pl, a, st) : launch_count_t<D, false, false>(ctx, pl, a, st);
}

// Run the count for B items of N packed points each; results: item_num[B] (device), per_origin (B == 1).
// force_split + hist (significance): SPLIT counters, and the finaliser histograms c_Q into hist[n_Q + 1].
ddks_status run_count(ddks_ctx* ctx, const float* packed, int d, int64_t B, int64_t n_P, int64_t n_Q,
                      int64_t o_begin, int64_t o_end, uint64_t* item_num, uint64_t* per_origin, cudaStream_t st,
                      bool force_split, unsigned long long* hist, bool wx, unsigned long long* best_key) {
    if (B == 1 && !wx && rank_applicable(ctx, d, n_P, n_Q, force_split))  // the rank-lane count (ddks_rank.cuh)
        return run_count_rank(ctx, packed, d, n_P, n_Q, o_begin, o_end, item_num, per_origin, st, best_key,
                              force_split || !diff_counters_ok(n_P, n_Q), hist);
    const int64_t N = n_P + n_Q;
    const uint64_t g = gcd_u64((uint64_t)n_P, (uint64_t)n_Q);
    const uint64_t a_ = (uint64_t)n_Q / g, b_ = (uint64_t)n_P / g;
    // DIFF counters hold c_P*a - c_Q*b: a 16-bit half stays in int16 over W <= 32767/max(a,b) points, and the
    // int32 total |value| <= n_P*n_Q/g must fit int32. Otherwise SPLIT: c_P and c_Q separately, W = 32767.
    const uint64_t mab = std::max(a_, b_);
    const bool split = force_split || mab > 32767 / 4096 || (uint64_t)n_P * a_ >= 0x7fffffffull || (uint64_t)n_Q * b_ >= 0x7fffffffull;
    const int64_t window = split ? 32767 : (int64_t)(32767 / mab);
    CountPlan pl{B, (int32_t)N, (int32_t)n_P, (int32_t)o_begin, (int32_t)o_end, n_P, n_Q, split, window};
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
    a.best_key = B == 1 ? best_key : nullptr;
    if (B > 65535) {  // grid.z limit: run the items in chunks
        for (int64_t b0 = 0; b0 < B; b0 += 65535) {
            const int64_t nb = std::min<int64_t>(65535, B - b0);
            ddks_status s = run_count(ctx, packed + b0 * N * pad_dim(d), d, nb, n_P, n_Q, o_begin, o_end,
                                      item_num + b0, nullptr, st, force_split, hist ? hist + b0 * (n_Q + 1) : nullptr,
                                      wx);
            if (s) return s;
        }
        return DDKS_OK;
    }
    switch (d) {
        case 1: return launch_count_d<1>(ctx, pl, a, st, wx);
        case 2: return launch_count_d<2>(ctx, pl, a, st, wx);
        case 3: return launch_count_d<3>(ctx, pl, a, st, wx);
        case 4: return launch_count_d<4>(ctx, pl, a, st, wx);
        case 5: return launch_count_d<5>(ctx, pl, a, st, wx);
        case 6: return launch_count_d<6>(ctx, pl, a, st, wx);
        case 7: return launch_count_d<7>(ctx, pl, a, st, wx);
        case 8: return launch_count_d<8>(ctx, pl, a, st, wx);
    }
    return fail(ctx, DDKS_ERR_DIM_UNSUPPORTED, "d=%d", d);
}

// Stable LSD radix sort of nseg segments of N 64-bit keys each, 8-bit digits from shift_begin up to bit 63;
// src and dst ping-pong; *sorted receives the buffer holding the result. hist: nseg * tiles * 256 uint32.
ddks_status radix_sort_keys(ddks_ctx* ctx, uint64_t* src, uint64_t* dst, int64_t N, int nseg, int shift_begin,
                            uint32_t* hist, cudaStream_t st, uint64_t** sorted) {
    const int tiles = (int)((N + ddks::RS_TILE - 1) / ddks::RS_TILE);
    for (int shift = shift_begin; shift < 64; shift += 8) {
        ddks::k_rs_hist<<<nseg * tiles, ddks::RS_T, 0, st>>>(src, N, tiles, shift, hist);
        ddks::k_rs_scan<<<nseg, 256 * ddks::RS_SCAN_PARTS, 0, st>>>(hist, tiles);
        ddks::k_rs_scatter<<<nseg * tiles, ddks::RS_T, 0, st>>>(src, dst, N, tiles, shift, hist);
        CHECK_LAUNCH();
        ctx->launches += 3;
        std::swap(src, dst);
    }
    *sorted = src;
    return DDKS_OK;
}

// DIFF counters fit (|c_P a - c_Q b| stays in int32 and the int16 window is >= 4096 points); else SPLIT
bool diff_counters_ok(int64_t n_P, int64_t n_Q) {
    const uint64_t g = gcd_u64((uint64_t)n_P, (uint64_t)n_Q);
    const uint64_t a_ = (uint64_t)n_Q / g, b_ = (uint64_t)n_P / g;
    return !(std::max(a_, b_) > 32767 / 4096 || (uint64_t)n_P * a_ >= 0x7fffffffull || (uint64_t)n_Q * b_ >= 0x7fffffffull);
}

bool x0_applicable(ddks_ctx* ctx, int d, int64_t n_P, int64_t n_Q, bool force_split) {
    if (ctx->flags & DDKS_FLAG_NO_X0) return false;
    // the sort pays for itself once the O(N^2) count dominates; DDKS_FLAG_FORCE_X0 (tests) lowers the bar. Crossover
    // (microbench/kd_threshold.py, profiles/r2_kd_midN_bucket.txt): radix-sorted kd at N ~ 60k-75k for d = 2..8; with
    // the mid-N bucket sort (single rank) at N ~ 40k for d = 3..8 (N = 40k: d = 3 1.05x, d = 4 1.05x, d = 5 1.04x,
    // d = 8 1.13x; N = 20k: 0.72-0.93x)
    // With the cluster ordering (round 2, second session; profiles/r2b_kd_threshold.txt): d = 8 pays from N = 20 000
    // (1.03x, 1.12x at 30 000), d = 3 from ~30 000 (1.15x), d = 4..6 only from ~40 000 (1.00-1.06x)
    // the rank-lane count beats the kd ordering at d = 8 (and is position-ordered: no sort)
    if (!(ctx->flags & DDKS_FLAG_FORCE_X0) && rank_applicable(ctx, d, n_P, n_Q, force_split)) return false;
    const bool single = ctx->world == 1;
    const int64_t mid = d >= 8 ? 20000 : (d == 3 ? 28000 : 40000);
    const int64_t min_n = (ctx->flags & DDKS_FLAG_FORCE_X0) ? 2 : (single && d >= 3 ? mid : 80000);
    return d >= 2 && d <= 8 && n_P + n_Q >= min_n;
}

ddks_status run_count_kd(ddks_ctx* ctx, const float* packed, int d, int64_t n_P, int64_t n_Q, int sw, int sr,
                         uint64_t* item_num, uint64_t* per_origin, cudaStream_t st, bool split,
                         unsigned long long* hist, unsigned long long* best_key) {
    switch (d) {
#define KD_CASE(D) case D: return run_count_kd_d<D>(ctx, packed, n_P, n_Q, sw, sr, item_num, per_origin, st, split, hist, best_key);
        KD_CASE(2) KD_CASE(3) KD_CASE(4) KD_CASE(5) KD_CASE(6) KD_CASE(7) KD_CASE(8)
#undef KD_CASE
    }
    return fail(ctx, DDKS_ERR_DIM_UNSUPPORTED, "kd mode d=%d", d);
}

bool argmax_key_fits(int64_t n_P, int64_t n_Q) {
    if (getenv("DDKS_NO_KEY")) return false;  // TEST ONLY: per-origin nums + k_argmax for any size
    const uint64_t g = gcd_u64((uint64_t)n_P, (uint64_t)n_Q);
    return (double)n_P * (double)n_Q / (double)g < 8589934592.0;  // num / g < 2^33: the packed key fits 64 bits
}

// One statistic (B == 1) over the origin shard [ob, oe) of this rank: count (kd-ordered when it applies, else
// position-ordered) into dres->num and, unless export_per (debug export of per-origin nums for [ob, oe)), this rank's
// argmax candidate: fused into the count kernel as the packed key dres->key when it fits (argmax_key_fits), else
// per-origin nums + k_argmax into dres->arg. No collective unless reduce_num_first (significance: the global num is
// all-reduced before the k_argmax path matches against it). split/hist: significance.
ddks_status count_statistic(ddks_ctx* ctx, const float* packed, int d, int64_t n_P, int64_t n_Q, int64_t ob,
                            int64_t oe, int sw, int sr, DevResult* dres, bool export_per, bool split,
                            unsigned long long* hist, cudaStream_t st, uint64_t** per_out, bool reduce_num_first) {
    const int64_t N = n_P + n_Q;
    ddks_status s;
    const bool use_key = !export_per && argmax_key_fits(n_P, n_Q);
    unsigned long long* key = use_key ? &dres->key : nullptr;
    const bool x0 = !export_per && x0_applicable(ctx, d, n_P, n_Q, split);
    *per_out = nullptr;
    ctx->rank_lanes = 0;  // set by run_count_rank when the rank-lane count runs
    if (x0) {
        // origins are positions of the kd order; per-origin nums (k_argmax path only) land in pooled order in per[N]
        uint64_t* per = nullptr;
        if (!use_key) {
            if ((s = ensure(ctx, ctx->per_origin, (size_t)N * 8))) return s;
            per = (uint64_t*)ctx->per_origin.p;
            CU(cudaMemsetAsync(per, 0, (size_t)N * 8, st));
        }
        *per_out = per;
        // SPLIT counters when the significance needs c_Q or DIFF counters would overflow (as in run_count)
        const bool sp = split || !diff_counters_ok(n_P, n_Q);
        if ((s = run_count_kd(ctx, packed, d, n_P, n_Q, sw, sr, (uint64_t*)&dres->num, per, st, sp, hist, key))) return s;
        if (use_key) return DDKS_OK;
        if (ctx->comm && reduce_num_first) NC(ncclAllReduce(&dres->num, &dres->num, 1, ncclUint64, ncclMax, ctx->comm, st));
        ddks::k_argmax<<<(int)std::min<int64_t>((N + 255) / 256, 148 * 4), 256, 0, st>>>(
            per, N, 0, (const uint64_t*)&dres->num, &dres->arg);
        CHECK_LAUNCH();
        ctx->launches++;
        return DDKS_OK;
    }
    ctx->kd_levels = 0;
    ctx->rank_lanes = 0;  // set by run_count_rank when the rank-lane count runs
    uint64_t* per = nullptr;
    if (!use_key) {
        if ((s = ensure(ctx, ctx->per_origin, (size_t)std::max<int64_t>(oe - ob, 1) * 8))) return s;
        per = (uint64_t*)ctx->per_origin.p;
    }
    *per_out = per;
    if (oe > ob && (s = run_count(ctx, packed, d, 1, n_P, n_Q, ob, oe, (uint64_t*)&dres->num, per, st, split, hist,
                                  false, key)))
        return s;
    if (export_per || use_key) return DDKS_OK;
    if (ctx->comm && reduce_num_first) NC(ncclAllReduce(&dres->num, &dres->num, 1, ncclUint64, ncclMax, ctx->comm, st));
    if (oe > ob) {
        ddks::k_argmax<<<(int)std::min<int64_t>((oe - ob + 255) / 256, 148 * 4), 256, 0, st>>>(
            per, oe - ob, ob, (const uint64_t*)&dres->num, &dres->arg);
        CHECK_LAUNCH();
        ctx->launches++;
    }
    return DDKS_OK;
}

// A rank's device result block -> its host record (decodes the packed argmax key when the fused path ran).
ddks_rank_record decode_record(const DevResult& r, int64_t n_P, int64_t n_Q, bool use_key) {
    ddks_rank_record o{};
    o.flags = r.flag;
    if (use_key) {
        const uint64_t g = gcd_u64((uint64_t)n_P, (uint64_t)n_Q);
        o.num = (r.key >> 31) * g;
        o.argmax_origin = r.key ? (int64_t)(0x7fffffffull - (r.key & 0x7fffffffull)) : -1;
    } else {
        o.num = r.num;
        o.argmax_origin = r.arg == ~0ull ? -1 : (int64_t)r.arg;
    }
    return o;
}

ddks_status launch_pack(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int d, int64_t B,
                        float* dst, uint32_t* flag, cudaStream_t st) {
    const int64_t total = B * (n_P + n_Q);
    if (total == 0) return DDKS_OK;
    const int threads = 256;
    const int blocks = (int)std::min<int64_t>((total + threads - 1) / threads, 148 * 8);
    ddks::k_pack<<<blocks, threads, 0, st>>>(P, n_P, Q, n_Q, d, B, dst, pad_dim(d),
                                            (ctx->flags & DDKS_FLAG_NO_VALIDATE) ? 0 : 1, flag);
    CHECK_LAUNCH();
    ctx->launches++;
    return DDKS_OK;
}

// Batches of small items (n_P, n_Q <= 1024, d >= 2): pack every label run in near-x_0 order (k_pack_sorted) so the
// count can decide bit 0 per warp (*wx = true); otherwise the plain pack.
ddks_status launch_pack_batch(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int d,
                              int64_t B, float* dst, uint32_t* flag, cudaStream_t st, bool* wx) {
    *wx = d >= 2 && n_P <= ddks::KPS_T * ddks::KPS_R && n_Q <= ddks::KPS_T * ddks::KPS_R && B <= 0x7fffffff &&
          !(ctx->flags & (DDKS_FLAG_TIES_GT | DDKS_FLAG_NO_X0));
    if (!*wx) return launch_pack(ctx, P, n_P, Q, n_Q, d, B, dst, flag, st);
    ddks::k_pack_sorted<<<dim3((unsigned)B, 2), ddks::KPS_T, 0, st>>>(P, n_P, Q, n_Q, d, dst, pad_dim(d),
                                                                      !(ctx->flags & DDKS_FLAG_NO_VALIDATE), flag);
    CHECK_LAUNCH();
    ctx->launches++;
    return DDKS_OK;
}

// Label-invariant permutation null (NEXT-2): labels + validation, then one classification per pair for J perms.
template <int D, int F>
ddks_status launch_perm_df(ddks_ctx* ctx, const float* pooled_packed, const int32_t* perms, int64_t n_perm,
                           int64_t n_P, int64_t n_Q, uint64_t* nums, uint32_t* flag, cudaStream_t st) {
    using G = ddks::PermGeo<D, F>;
    const bool gt = (ctx->flags & DDKS_FLAG_TIES_GT) != 0;
    auto kern = gt ? ddks::k_perm_count<D, true, F> : ddks::k_perm_count<D, false, F>;
    static std::atomic<bool> attr[kMaxDevices][2] = {};
    if (ctx->device >= kMaxDevices) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "device index %d >= %d", ctx->device, kMaxDevices);
    if (!attr[ctx->device][gt].load(std::memory_order_acquire)) {
        CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM_BYTES));
        attr[ctx->device][gt].store(true, std::memory_order_release);
    }
    const int64_t N = n_P + n_Q;
    const int64_t chunks = (n_perm + G::J - 1) / G::J;
    const int64_t words = (N + 31) / 32;
    // [chunks][chunk_words] increment words; rows padded to 16 bytes (+16: the last bulk copy rounds up to 16)
    const int64_t chunk_words = (N * G::JW + 3) & ~int64_t(3);
    const size_t lab_bytes = (size_t)chunks * chunk_words * 4 + 16;
    ddks_status s;
    if ((s = ensure(ctx, ctx->labels, lab_bytes))) return s;
    if ((s = ensure(ctx, ctx->bitmap, (size_t)n_perm * words * 4))) return s;
    CU(cudaMemsetAsync(ctx->labels.p, 0, lab_bytes, st));
    CU(cudaMemsetAsync(ctx->bitmap.p, 0, (size_t)n_perm * words * 4, st));
    const int64_t tot = n_perm * N;
    const int blocks = (int)std::min<int64_t>((tot + 255) / 256, 148 * 8);
    ddks::k_labels<<<blocks, 256, 0, st>>>(perms, n_perm, N, n_P, G::J, G::JW, F, chunk_words,
                                           (uint32_t*)ctx->labels.p, (uint32_t*)ctx->bitmap.p, flag);
    CHECK_LAUNCH();
    ctx->launches++;
    const uint64_t g = gcd_u64((uint64_t)n_P, (uint64_t)n_Q);
    ddks::PermArgs pa{};
    pa.pts = pooled_packed;
    pa.labels = (const uint32_t*)ctx->labels.p;
    pa.chunk_words = chunk_words;
    pa.N = (int32_t)N;
    pa.n_perm = (int32_t)n_perm;
    pa.a = (uint32_t)((uint64_t)n_Q / g);
    pa.b = (uint32_t)((uint64_t)n_P / g);
    pa.g = g;
    pa.num = nums;
    pa.clk = nullptr;
    dim3 grid((unsigned)chunks, (unsigned)((N + G::T - 1) / G::T));
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
        if ((s = ensure_prof(ctx))) return s;
        pa.clk = (unsigned long long*)ctx->prof_clk.p;
    }
    kern<<<grid, G::T, G::SMEM_BYTES, st>>>(pa);
    CHECK_LAUNCH();
    ctx->launches++;
    if (ev.first) {
        CU(record_event(ev.second, st));
        ctx->ev_pending.push_back(ev);
        ctx->ev_recycle.push_back(1);
        // classifications actually performed: each pair is classified once per chunk of J permutations
        ctx->ev_pairs.push_back((uint64_t)chunks * (uint64_t)N * (uint64_t)N);
    }
    return DDKS_OK;
}

template <int D>
ddks_status launch_perm_d(ddks_ctx* ctx, const float* pooled_packed, const int32_t* perms, int64_t n_perm,
                          int64_t n_P, int64_t n_Q, uint64_t* nums, uint32_t* flag, cudaStream_t st) {
    // 10-bit label counters (three permutations per word) whenever c_P' <= n_P fits them
    if (n_P <= 1023) return launch_perm_df<D, 10>(ctx, pooled_packed, perms, n_perm, n_P, n_Q, nums, flag, st);
    return launch_perm_df<D, 16>(ctx, pooled_packed, perms, n_perm, n_P, n_Q, nums, flag, st);
}

// Tensor-core null (ddks_perm_mma.cuh): label images + validation, then the one-hot x label contraction per
// 128 x 256 tile. pooled_packed must hold ceil(N / PM_KB) * PM_KB rows (the tail zeroed by the caller).
template <int D>
ddks_status launch_perm_mma_d(ddks_ctx* ctx, const float* pooled_packed, const int32_t* perms, int64_t n_perm,
                              int64_t n_P, int64_t n_Q, uint64_t* nums, uint32_t* flag, cudaStream_t st) {
    using G = ddks::PermMmaGeo<D>;
    const bool gt = (ctx->flags & DDKS_FLAG_TIES_GT) != 0;
    auto kern = gt ? ddks::k_perm_mma<D, true> : ddks::k_perm_mma<D, false>;
    static std::atomic<bool> attr[kMaxDevices][2] = {};
    if (!attr[ctx->device][gt].load(std::memory_order_acquire)) {
        CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM_BYTES));
        attr[ctx->device][gt].store(true, std::memory_order_release);
    }
    const int64_t N = n_P + n_Q;
    const int64_t kblocks = (N + ddks::PM_KB - 1) / ddks::PM_KB;
    const int64_t n_tiles = (n_perm + ddks::PM_N - 1) / ddks::PM_N;
    const size_t bimg_bytes = (size_t)n_tiles * kblocks * ddks::PM_B_BYTES;
    const int64_t words = (N + 31) / 32;
    ddks_status s;
    if ((s = ensure(ctx, ctx->labels, bimg_bytes))) return s;
    if ((s = ensure(ctx, ctx->bitmap, (size_t)n_perm * words * 4))) return s;
    CU(cudaMemsetAsync(ctx->labels.p, 0, bimg_bytes, st));
    CU(cudaMemsetAsync(ctx->bitmap.p, 0, (size_t)n_perm * words * 4, st));
    const int64_t tot = n_perm * N;
    ddks::k_labels_mma<<<(int)std::min<int64_t>((tot + 255) / 256, 148 * 8), 256, 0, st>>>(
        perms, n_perm, N, n_P, (int)kblocks, (uint8_t*)ctx->labels.p, (uint32_t*)ctx->bitmap.p, flag);
    CHECK_LAUNCH();
    ctx->launches++;
    const uint64_t g = gcd_u64((uint64_t)n_P, (uint64_t)n_Q);
    ddks::PermMmaArgs pa{};
    pa.pts = pooled_packed;
    pa.bimg = (const uint8_t*)ctx->labels.p;
    pa.N = (int32_t)N;
    pa.n_perm = (int32_t)n_perm;
    pa.k_blocks = (int32_t)kblocks;
    pa.a = (uint32_t)((uint64_t)n_Q / g);
    pa.b = (uint32_t)((uint64_t)n_P / g);
    pa.g = g;
    pa.num = nums;
    pa.clk = nullptr;
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
        if ((s = ensure_prof(ctx))) return s;
        pa.clk = (unsigned long long*)ctx->prof_clk.p;
    }
    const dim3 grid((unsigned)((N + G::OPT - 1) / G::OPT), (unsigned)n_tiles);
    kern<<<grid, ddks::PM_THREADS, G::SMEM_BYTES, st>>>(pa);
    CHECK_LAUNCH();
    ctx->launches++;
    if (ev.first) {
        CU(record_event(ev.second, st));
        ctx->ev_pending.push_back(ev);
        ctx->ev_recycle.push_back(1);
        // pair classifications performed: every (origin, point) pair once per tile column group of 256 permutations
        ctx->ev_pairs.push_back((uint64_t)n_tiles * (uint64_t)N * (uint64_t)N);
    }
    return DDKS_OK;
}

// the tensor-core null applies: d <= 7, the label path's N <= 65535 (exact fp32 sums, u32 column maxima)
bool perm_mma_applies(ddks_ctx* ctx, int d, int64_t N) {
    return d <= 7 && N <= 65535 && !getenv("DDKS_NO_MMA") && !(ctx->flags & DDKS_FLAG_PERM_GATHER);
}

ddks_status launch_perm_mma(ddks_ctx* ctx, int d, const float* pooled_packed, const int32_t* perms, int64_t n_perm,
                            int64_t n_P, int64_t n_Q, uint64_t* nums, uint32_t* flag, cudaStream_t st) {
    switch (d) {
#define PMMA_CASE(D) case D: return launch_perm_mma_d<D>(ctx, pooled_packed, perms, n_perm, n_P, n_Q, nums, flag, st);
        PMMA_CASE(1) PMMA_CASE(2) PMMA_CASE(3) PMMA_CASE(4) PMMA_CASE(5) PMMA_CASE(6) PMMA_CASE(7)
#undef PMMA_CASE
    }
    return fail(ctx, DDKS_ERR_DIM_UNSUPPORTED, "tensor-core null d=%d", d);
}

ddks_status launch_perm(ddks_ctx* ctx, int d, const float* pooled_packed, const int32_t* perms, int64_t n_perm,
                        int64_t n_P, int64_t n_Q, uint64_t* nums, uint32_t* flag, cudaStream_t st) {
    switch (d) {
        case 1: return launch_perm_d<1>(ctx, pooled_packed, perms, n_perm, n_P, n_Q, nums, flag, st);
        case 2: return launch_perm_d<2>(ctx, pooled_packed, perms, n_perm, n_P, n_Q, nums, flag, st);
        case 3: return launch_perm_d<3>(ctx, pooled_packed, perms, n_perm, n_P, n_Q, nums, flag, st);
        case 4: return launch_perm_d<4>(ctx, pooled_packed, perms, n_perm, n_P, n_Q, nums, flag, st);
        case 5: return launch_perm_d<5>(ctx, pooled_packed, perms, n_perm, n_P, n_Q, nums, flag, st);
        case 6: return launch_perm_d<6>(ctx, pooled_packed, perms, n_perm, n_P, n_Q, nums, flag, st);
        case 7: return launch_perm_d<7>(ctx, pooled_packed, perms, n_perm, n_P, n_Q, nums, flag, st);
        case 8: return launch_perm_d<8>(ctx, pooled_packed, perms, n_perm, n_P, n_Q, nums, flag, st);
    }
    return fail(ctx, DDKS_ERR_DIM_UNSUPPORTED, "d=%d", d);
}

ddks_status ensure_host(ddks_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->host_pinned_bytes) return DDKS_OK;
    if (ctx->host_pinned) cudaFreeHost(ctx->host_pinned);
    ctx->alloc_epoch++;
    ctx->host_pinned = nullptr;
    ctx->host_pinned_bytes = 0;
    CU(cudaMallocHost(&ctx->host_pinned, bytes));
    ctx->host_pinned_bytes = bytes;
    return DDKS_OK;
}

ddks_status prof_begin(ddks_ctx* ctx, cudaStream_t st, std::pair<cudaEvent_t, cudaEvent_t>* ev) {
    *ev = {nullptr, nullptr};
    if (!(ctx->flags & DDKS_FLAG_PROFILE)) return DDKS_OK;
    if (!ctx->ev_free.empty()) {
        *ev = ctx->ev_free.back();
        ctx->ev_free.pop_back();
    } else {
        CU(cudaEventCreate(&ev->first));
        CU(cudaEventCreate(&ev->second));
    }
    CU(record_event(ev->first, st));
    return DDKS_OK;
}

ddks_status prof_end(ddks_ctx* ctx, cudaStream_t st, const std::pair<cudaEvent_t, cudaEvent_t>& ev, uint64_t units) {
    if (!ev.first) return DDKS_OK;
    CU(record_event(ev.second, st));
    ctx->ev_pending.push_back(ev);
    ctx->ev_recycle.push_back(1);
    ctx->ev_pairs.push_back(units);
    return DDKS_OK;
}

// After a stream sync: fold the pending count-kernel events into the profile totals.
ddks_status collect_profile(ddks_ctx* ctx) {
    for (size_t i = 0; i < ctx->ev_pending.size(); ++i) {
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, ctx->ev_pending[i].first, ctx->ev_pending[i].second));
        ctx->prof_ms += ms;
        ctx->prof_launches += 1;
        ctx->prof_pairs += ctx->ev_pairs[i];
        if (i >= ctx->ev_recycle.size() || ctx->ev_recycle[i]) ctx->ev_free.push_back(ctx->ev_pending[i]);
    }
    ctx->ev_pending.clear();
    ctx->ev_pairs.clear();
    ctx->ev_recycle.clear();
    return DDKS_OK;
}

ddks_status bind_device(ddks_ctx* ctx) {
    CU(cudaSetDevice(ctx->device));
    return DDKS_OK;
}

// Items sharded contiguously over the ranks (ddks_shard_range): ONE ncclAllGather of a padded per-rank record --
// this rank's slice of each of the n_arr device arrays dev[k][total] (8-byte elements), each padded to chunk = rank 0's
// (largest) shard, then this rank's flag word -- into ctx->gather, copied to host hbuf[world * stride] (stride =
// n_arr * chunk + 1). The caller unpads it with ddks_unpad_items (host), which also ORs the flags.
ddks_status gather_items(ddks_ctx* ctx, uint64_t* const* dev, int n_arr, int64_t total, const uint32_t* dflag,
                         cudaStream_t st, uint64_t* hbuf) {
    int64_t b0, b1;
    ddks_shard_range(total, ctx->world, 0, &b0, &b1);
    const int64_t chunk = b1 - b0;
    const int64_t stride = chunk * n_arr + 1;
    ddks_status s = ensure(ctx, ctx->gather, (size_t)(ctx->world + 1) * stride * 8);
    if (s) return s;
    uint64_t* all = (uint64_t*)ctx->gather.p;
    uint64_t* send = all + (int64_t)ctx->world * stride;
    int64_t mb, me;
    ddks_shard_range(total, ctx->world, ctx->rank, &mb, &me);
    CU(cudaMemsetAsync(send, 0, (size_t)stride * 8, st));
    for (int k = 0; k < n_arr; ++k)
        if (me > mb) CU(cudaMemcpyAsync(send + k * chunk, dev[k] + mb, (size_t)(me - mb) * 8, cudaMemcpyDeviceToDevice, st));
    CU(cudaMemcpyAsync(send + n_arr * chunk, dflag, 4, cudaMemcpyDeviceToDevice, st));
    NC(ncclAllGather(send, all, (size_t)stride, ncclUint64, ctx->comm, st));
    CU(cudaMemcpyAsync(hbuf, all, (size_t)ctx->world * stride * 8, cudaMemcpyDeviceToHost, st));
    return DDKS_OK;
}

int64_t gather_stride(int64_t total, int world, int n_arr) {
    return (total / world + (total % world ? 1 : 0)) * n_arr + 1;
}

// a graph may read this input at replay time: device (or managed) memory, or page-locked host memory
bool graph_input_ok(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged || a.type == cudaMemoryTypeHost;
}

// environment overrides (tuning / test knobs) change the plan: a graph captured under other values is not reused
bool env_overrides() {
    return getenv("DDKS_KD") || getenv("DDKS_SEGS") || getenv("DDKS_KD_SHUFFLE") || getenv("DDKS_NO_KEY") ||
           getenv("DDKS_GRIDY") || getenv("DDKS_NO_SMALL") || getenv("DDKS_KD_RADIX") || getenv("DDKS_NO_MMA") ||
           getenv("DDKS_PERM_GROUP") || getenv("DDKS_KD_FUSED") || getenv("DDKS_RANK_SK");
}

void drop_call_graph(ddks_ctx* ctx, ddks_ctx::CallGraph& cg) {
    if (cg.exec) cudaGraphExecDestroy(cg.exec);
    cg.exec = nullptr;
    cg.key.clear();
    for (auto& e : cg.evs) ctx->ev_free.push_back(e);
    cg.evs.clear();
    cg.ev_pairs.clear();
}

void launch_call_graph(ddks_ctx* ctx, ddks_ctx::CallGraph& cg, cudaStream_t st, cudaError_t* e) {
    *e = cudaGraphLaunch(cg.exec, st);
    ctx->launches += cg.launches;
    for (size_t i = 0; i < cg.evs.size(); ++i) {
        ctx->ev_pending.push_back(cg.evs[i]);
        ctx->ev_pairs.push_back(cg.ev_pairs[i]);
        ctx->ev_recycle.push_back(0);
    }
}

}  // namespace ddks_host

using namespace ddks_host;

// ===================================================================================================== C ABI
extern "C" {

const char* ddks_version(void) { return DDKS_VERSION; }

ddks_status ddks_shard_range(int64_t total, int world, int rank, int64_t* begin, int64_t* end) {
    if (!begin || !end || total < 0 || world < 1 || rank < 0 || rank >= world) return DDKS_ERR_INVALID_ARGUMENT;
    const int64_t base = total / world, rem = total % world;
    *begin = rank * base + std::min<int64_t>(rank, rem);
    *end = *begin + base + (rank < rem ? 1 : 0);
    return DDKS_OK;
}

ddks_status ddks_combine_records(const ddks_rank_record* recs, int world, ddks_rank_record* out) {
    if (!recs || !out || world < 1) return DDKS_ERR_INVALID_ARGUMENT;
    ddks_rank_record r{0ull, -1, 0u, 0u};
    for (int i = 0; i < world; ++i) {
        r.flags |= recs[i].flags;
        if (recs[i].num > r.num) r.num = recs[i].num;
    }
    for (int i = 0; i < world; ++i)
        if (recs[i].num == r.num && recs[i].argmax_origin >= 0 &&
            (r.argmax_origin < 0 || recs[i].argmax_origin < r.argmax_origin))
            r.argmax_origin = recs[i].argmax_origin;
    *out = r;
    return DDKS_OK;
}

ddks_status ddks_unpad_items(const uint64_t* gathered, int64_t total, int world, int n_arr, uint64_t* out,
                             uint32_t* flags) {
    if (!gathered || !out || total < 0 || world < 1 || n_arr < 1) return DDKS_ERR_INVALID_ARGUMENT;
    int64_t b0, b1;
    ddks_shard_range(total, world, 0, &b0, &b1);
    const int64_t chunk = b1 - b0, stride = chunk * n_arr + 1;
    uint32_t f = 0;
    for (int r = 0; r < world; ++r) {
        int64_t rb, re;
        ddks_shard_range(total, world, r, &rb, &re);
        const uint64_t* rec = gathered + (int64_t)r * stride;
        for (int k = 0; k < n_arr; ++k)
            for (int64_t i = rb; i < re; ++i) out[(int64_t)k * total + i] = rec[(int64_t)k * chunk + (i - rb)];
        f |= (uint32_t)rec[(int64_t)n_arr * chunk];
    }
    if (flags) *flags = f;
    return DDKS_OK;
}

ddks_status ddks_get_nccl_id(void* out_128_bytes) {
    ddks_ctx* ctx = nullptr;
    if (!out_128_bytes) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "null id buffer");
    ncclUniqueId id;
    NC(ncclGetUniqueId(&id));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    memcpy(out_128_bytes, &id, 128);
    return DDKS_OK;
}

ddks_status ddks_create(ddks_ctx** out, int device, int world, int rank, const void* nccl_id, uint32_t flags) {
    ddks_ctx* ctx = nullptr;
    if (!out) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "null out");
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "bad world/rank");
    if ((world == 1) != (nccl_id == nullptr))
        return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "nccl_id must be NULL iff world == 1");
    if (flags & ~(DDKS_FLAG_NO_VALIDATE | DDKS_FLAG_TIES_GT | DDKS_FLAG_FORCE_DIRECT | DDKS_FLAG_PROFILE | DDKS_FLAG_PERM_GATHER | DDKS_FLAG_NO_X0 | DDKS_FLAG_FORCE_X0 | DDKS_FLAG_RDKS_FULL_SORT | DDKS_FLAG_KD_LEVELS(7) | DDKS_FLAG_NCCL_SELF | DDKS_FLAG_NO_GRAPH | DDKS_FLAG_NO_RANK | DDKS_FLAG_FORCE_RANK)) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "bad flags");
    int ndev = 0;
    CU(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "device %d of %d", device, ndev);
    CU(cudaSetDevice(device));
    ctx = new ddks_ctx();
    ctx->device = device;
    ctx->world = world;
    ctx->rank = rank;
    ctx->flags = flags;
    if (world > 1 || (flags & DDKS_FLAG_NCCL_SELF)) {
        // world > 1: the harness's id; NCCL_SELF (tests): a one-rank communicator of our own, so every collective
        // of the multi-GPU path runs through NCCL on a single device
        ncclUniqueId id;
        if (world > 1) {
            memcpy(&id, nccl_id, sizeof id);
        } else {
            ncclResult_t g = ncclGetUniqueId(&id);
            if (g != ncclSuccess) {
                fail(nullptr, DDKS_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(g));
                delete ctx;
                return DDKS_ERR_NCCL;
            }
        }
        ncclResult_t r = ncclCommInitRank(&ctx->comm, world, id, rank);
        if (r != ncclSuccess) {
            fail(nullptr, DDKS_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
            delete ctx;
            return DDKS_ERR_NCCL;
        }
    }
    ddks_status s = ensure(ctx, ctx->res, sizeof(DevResult));
    if (!s) s = ensure_host(ctx, 4096);
    if (s) {
        g_create_err = ctx->err;
        ddks_destroy(ctx);
        return s;
    }
    *out = ctx;
    return DDKS_OK;
}

ddks_status ddks_destroy(ddks_ctx* ctx) {
    if (!ctx) return DDKS_OK;
    cudaSetDevice(ctx->device);
    if (ctx->comm) ncclCommDestroy(ctx->comm);
    if (ctx->sg_exec) cudaGraphExecDestroy(ctx->sg_exec);
    for (auto* cg : {&ctx->cg_batch, &ctx->cg_null, &ctx->cg_vdks, &ctx->cg_rdks})
        if (cg->exec) cudaGraphExecDestroy(cg->exec);
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    for (auto e : ctx->copy_evs) cudaEventDestroy(e);
    for (auto* v : {&ctx->ev_free, &ctx->sg_evs, &ctx->cg_batch.evs, &ctx->cg_null.evs, &ctx->cg_vdks.evs,
                    &ctx->cg_rdks.evs})
        for (auto& e : *v) {
            cudaEventDestroy(e.first);
            cudaEventDestroy(e.second);
        }
    for (size_t i = 0; i < ctx->ev_pending.size(); ++i)  // left pending only by a failed call
        if (i < ctx->ev_recycle.size() && ctx->ev_recycle[i]) {
            cudaEventDestroy(ctx->ev_pending[i].first);
            cudaEventDestroy(ctx->ev_pending[i].second);
        }
    for (DevBuf* b : {&ctx->raw_a, &ctx->raw_b, &ctx->raw_perm, &ctx->packed, &ctx->packed2, &ctx->pool_packed, &ctx->per_origin,
                      &ctx->accum, &ctx->gather, &ctx->item_num, &ctx->bitmap, &ctx->labels, &ctx->res, &ctx->sig_hist,
                      &ctx->sig_lf, &ctx->sig_scratch, &ctx->sig_table, &ctx->sig_contrib, &ctx->sig_part,
                      &ctx->vox_keys, &ctx->vox_cnt, &ctx->vox_S, &ctx->vox_fill, &ctx->vox_slab, &ctx->rd_keys, &ctx->rd_xn, &ctx->rd_k0,
                      &ctx->rd_k1, &ctx->rd_hist, &ctx->rd_tcnt, &ctx->rd_cnum, &ctx->x0_keys0,
                      &ctx->x0_keys1, &ctx->x0_hist, &ctx->x0_pts, &ctx->x0_perm, &ctx->x0_pts2,
                      &ctx->x0_perm2, &ctx->x0_boxes, &ctx->prof_clk, &ctx->rdb_cnt,
                      &ctx->rdb_pst, &ctx->rdb_coff, &ctx->rdb_fill, &ctx->rdb_clist, &ctx->rdb_csum, &ctx->rdb_bits,
                      &ctx->kdf_bar, &ctx->kdf_buf, &ctx->rank_v})
        if (b->p) cudaFree(b->p);
    if (ctx->host_pinned) cudaFreeHost(ctx->host_pinned);
    delete ctx;
    return DDKS_OK;
}

const char* ddks_last_error(const ddks_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

int64_t ddks_launch_count(const ddks_ctx* ctx) { return ctx ? ctx->launches : 0; }

int32_t ddks_kd_levels(const ddks_ctx* ctx) { return ctx ? ctx->kd_levels : 0; }

int32_t ddks_rank_lanes(const ddks_ctx* ctx) { return ctx ? ctx->rank_lanes : 0; }

ddks_status ddks_profile_read(ddks_ctx* ctx, double* count_ms, int64_t* launches, uint64_t* pairs) {
    if (!ctx) return DDKS_ERR_INVALID_ARGUMENT;
    ddks_status s = collect_profile(ctx);
    if (s) return s;
    if (count_ms) *count_ms = ctx->prof_ms;
    if (launches) *launches = ctx->prof_launches;
    if (pairs) *pairs = ctx->prof_pairs;
    ctx->prof_ms = 0.0;
    ctx->prof_launches = 0;
    ctx->prof_pairs = 0;
    return DDKS_OK;
}

ddks_status ddks_profile_clock(ddks_ctx* ctx, double* sm_mhz) {
    if (!ctx || !sm_mhz) return DDKS_ERR_INVALID_ARGUMENT;
    *sm_mhz = 0.0;
    if (!ctx->prof_clk.p) return DDKS_OK;
    // the probe totals accumulate on the device across calls (no per-call copy inside a timed region); read here
    CU(cudaSetDevice(ctx->device));
    CU(cudaDeviceSynchronize());
    unsigned long long c[2];
    CU(cudaMemcpy(c, ctx->prof_clk.p, 16, cudaMemcpyDeviceToHost));
    CU(cudaMemset(ctx->prof_clk.p, 0, 16));
    *sm_mhz = c[1] > 0 ? (double)c[0] / (double)c[1] * 1e3 : 0.0;
    return DDKS_OK;
}

ddks_status ddks_profile_work(ddks_ctx* ctx, uint64_t* compares) {
    if (!ctx || !compares) return DDKS_ERR_INVALID_ARGUMENT;
    *compares = 0;
    if (!ctx->prof_clk.p) return DDKS_OK;
    CU(cudaSetDevice(ctx->device));
    CU(cudaDeviceSynchronize());
    unsigned long long c = 0;
    CU(cudaMemcpy(&c, (unsigned long long*)ctx->prof_clk.p + 2, 8, cudaMemcpyDeviceToHost));
    CU(cudaMemset((unsigned long long*)ctx->prof_clk.p + 2, 0, 8));
    *compares = c;
    return DDKS_OK;
}

}  // extern "C"

// The fused small-N path (ddks_small.cuh) applies: single rank, whole statistic, N <= kSmallFusedN, DIFF counters whose
// int16 halves hold the whole point set (N * max(a, b) <= 32767, so the DSMEM word adds are exact).
constexpr int64_t kSmallFusedN = 8192;
static bool small_fused_applies(ddks_ctx* ctx, int64_t n_P, int64_t n_Q) {
    // DDKS_NO_SMALL and the FORCE_X0 / FORCE_DIRECT test flags keep the packed path reachable at small N
    if (ctx->comm || getenv("DDKS_NO_SMALL") || (ctx->flags & (DDKS_FLAG_FORCE_X0 | DDKS_FLAG_FORCE_DIRECT))) return false;
    const int64_t N = n_P + n_Q;
    if (N > kSmallFusedN || !diff_counters_ok(n_P, n_Q)) return false;
    const uint64_t g = gcd_u64((uint64_t)n_P, (uint64_t)n_Q);
    return (uint64_t)N * std::max((uint64_t)n_Q / g, (uint64_t)n_P / g) <= 32767;
}
static int64_t small_blocks(int64_t N) { return (N + ddks::SM_R * ddks::SM_T - 1) / (ddks::SM_R * ddks::SM_T); }

template <int D>
static ddks_status launch_small_d(ddks_ctx* ctx, const ddks::SmallArgs& a, int segs, int blocks, cudaStream_t st) {
    const bool gt = (ctx->flags & DDKS_FLAG_TIES_GT) != 0;
    auto kern = gt ? ddks::k_count_small<D, true> : ddks::k_count_small<D, false>;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3((unsigned)segs, (unsigned)blocks, 1);
    cfg.blockDim = dim3(ddks::SM_T, 1, 1);
    cfg.dynamicSmemBytes = ddks::SmallGeo<D>::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)segs;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    static std::atomic<bool> done[kMaxDevices][2] = {};
    if (!done[ctx->device][gt].load(std::memory_order_acquire)) {
        CU(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ddks::SmallGeo<D>::SMEM_BYTES));
        done[ctx->device][gt].store(true, std::memory_order_release);
    }
    CU(cudaLaunchKernelEx(&cfg, kern, a));
    ctx->launches++;
    return DDKS_OK;
}

// Enqueue the fused small-N statistic: one cluster launch whose leaders write per-origin-block records into the pinned
// host buffer (reduced by stat_impl after the sync). No result initialisation, no copy: the call is one graph node.
static ddks_status small_enqueue(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int32_t d,
                                 cudaStream_t st, void* host_rec = nullptr) {
    ddks_status s;
    const int64_t N = n_P + n_Q;
    const void *dP, *dQ;
    if ((s = stage_input(ctx, P, (size_t)n_P * d * 4, ctx->raw_a, st, &dP))) return s;
    if ((s = stage_input(ctx, Q, (size_t)n_Q * d * 4, ctx->raw_b, st, &dQ))) return s;
    const int64_t blocks = small_blocks(N);
    // the points split over a full cluster (8 CTAs, segments of whole warps' worth of rows): at N = 400 every CTA
    // counts 64 points for its 256 origins, latency rather than issue being the limit at this size
    const int64_t seg_points = std::max<int64_t>(32, (N + 8 * ddks::SM_MAX_CLUSTER - 1) / (8 * ddks::SM_MAX_CLUSTER) * 8);
    const int segs = (int)((N + seg_points - 1) / seg_points);
    const uint64_t g = gcd_u64((uint64_t)n_P, (uint64_t)n_Q);
    ddks::SmallArgs a{};
    a.P = (const float*)dP;
    a.Q = (const float*)dQ;
    a.n_P = (int32_t)n_P;
    a.N = (int32_t)N;
    a.seg_points = (int32_t)seg_points;
    a.incP = (uint32_t)((uint64_t)n_Q / g);
    a.incQ = 0u - (uint32_t)((uint64_t)n_P / g);
    a.gg = g;
    a.validate = (ctx->flags & DDKS_FLAG_NO_VALIDATE) ? 0 : 1;
    // the leaders write their records straight into the context's pinned host buffer (zero-copy: no D2H node)
    void* hdev = nullptr;
    CU(cudaHostGetDevicePointer(&hdev, host_rec ? host_rec : ctx->host_pinned, 0));
    a.out = (unsigned long long*)hdev;
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
        if ((s = ensure_prof(ctx))) return s;
        a.clk = (unsigned long long*)ctx->prof_clk.p;
    }
    ctx->kd_levels = 0;
    ctx->rank_lanes = 0;
    switch (d) {
#define SM_CASE(D) case D: s = launch_small_d<D>(ctx, a, segs, (int)blocks, st); break;
        SM_CASE(1) SM_CASE(2) SM_CASE(3) SM_CASE(4) SM_CASE(5) SM_CASE(6) SM_CASE(7) SM_CASE(8)
#undef SM_CASE
        default: return fail(ctx, DDKS_ERR_DIM_UNSUPPORTED, "d=%d", d);
    }
    if (s) return s;
    if (ev.first) {
        CU(record_event(ev.second, st));
        ctx->ev_pending.push_back(ev);
        ctx->ev_recycle.push_back(1);
        ctx->ev_pairs.push_back((uint64_t)N * (uint64_t)N);
    }
    return DDKS_OK;
}

extern "C" {

// Enqueue one statistic on st, ending with the D2H of the result record(s) into host_pinned (no sync): staging of host
// inputs, pack, count (+ fused argmax), and with world > 1 the ONE collective: the all-gather of every rank's 32-byte
// result record (host_pinned then holds world records, combined by ddks_combine_records after the sync). Everything
// here is stream-ordered, so it can be captured.
static ddks_status stat_enqueue(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int32_t d,
                                cudaStream_t st, int64_t ob, int64_t oe, uint64_t* per_origin_out, int sw, int sr,
                                bool small) {
    ddks_status s;
    const int64_t N = n_P + n_Q;
    const int DP = pad_dim(d);
    const bool export_mode = per_origin_out != nullptr;
    if (small) return small_enqueue(ctx, P, n_P, Q, n_Q, d, st);
    const void *dP, *dQ;
    if ((s = stage_input(ctx, P, (size_t)n_P * d * 4, ctx->raw_a, st, &dP))) return s;
    if ((s = stage_input(ctx, Q, (size_t)n_Q * d * 4, ctx->raw_b, st, &dQ))) return s;
    if ((s = ensure(ctx, ctx->packed, (size_t)N * DP * 4))) return s;
    const bool gather = ctx->comm && !export_mode;
    if (gather && (s = ensure(ctx, ctx->gather, (size_t)ctx->world * sizeof(DevResult)))) return s;
    DevResult* dres = (DevResult*)ctx->res.p;
    DevResult* hres = (DevResult*)ctx->host_pinned;
    *hres = DevResult{0ull, ~0ull, 0ull, 0u, 0u};  // re-written by the host before every graph replay as well
    CU(cudaMemcpyAsync(dres, hres, sizeof(DevResult), cudaMemcpyHostToDevice, st));
    float* packed = (float*)ctx->packed.p;
    if ((s = launch_pack(ctx, (const float*)dP, n_P, (const float*)dQ, n_Q, d, 1, packed, &dres->flag, st))) return s;
    uint64_t* per = nullptr;
    if ((s = count_statistic(ctx, packed, d, n_P, n_Q, ob, oe, sw, sr, dres, export_mode, false, nullptr, st, &per,
                             false)))
        return s;
    if (export_mode && oe > ob) {
        CU(cudaMemcpyAsync(per_origin_out, per, (size_t)(oe - ob) * 8, cudaMemcpyDefault, st));
    }
    if (gather) {
        static_assert(sizeof(DevResult) % 8 == 0, "record of uint64 words");
        NC(ncclAllGather(dres, ctx->gather.p, sizeof(DevResult) / 8, ncclUint64, ctx->comm, st));
        CU(cudaMemcpyAsync(hres, ctx->gather.p, (size_t)ctx->world * sizeof(DevResult), cudaMemcpyDeviceToHost, st));
    } else {
        CU(cudaMemcpyAsync(hres, dres, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
    }
    return DDKS_OK;
}


static void drop_stat_graph(ddks_ctx* ctx) {
    if (ctx->sg_exec) cudaGraphExecDestroy(ctx->sg_exec);
    ctx->sg_exec = nullptr;
    ctx->sg_key = ddks_ctx::StatKey{};
    // the graph's event pairs: no longer pending (every call collects before returning), so they are free again
    for (auto& e : ctx->sg_evs) ctx->ev_free.push_back(e);
    ctx->sg_evs.clear();
    ctx->sg_ev_pairs.clear();
}

// Capture stat_enqueue on the context's capture stream into ctx->sg_exec. *ok = false (and no error) when the capture
// or instantiation is refused or the workspace moved meanwhile; the caller then runs the call uncaptured.
static ddks_status stat_capture(ddks_ctx* ctx, const ddks_ctx::StatKey& key, const float* P, int64_t n_P,
                                const float* Q, int64_t n_Q, int32_t d, int64_t ob, int64_t oe, int sw, int sr,
                                bool* ok) {
    *ok = false;
    drop_stat_graph(ctx);
    if (!ctx->cap_stream) CU(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
    const size_t ev0 = ctx->ev_pending.size();
    const int64_t l0 = ctx->launches;
    CU(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeRelaxed));
    const ddks_status s = stat_enqueue(ctx, P, n_P, Q, n_Q, d, ctx->cap_stream, ob, oe, nullptr, sw, sr,
                                       small_fused_applies(ctx, n_P, n_Q));
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(ctx->cap_stream, &g);
    // the events recorded during the capture are graph nodes (not executed yet): they belong to the graph
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> evs(ctx->ev_pending.begin() + ev0, ctx->ev_pending.end());
    std::vector<uint64_t> pairs(ctx->ev_pairs.begin() + ev0, ctx->ev_pairs.end());
    ctx->ev_pending.resize(ev0);
    ctx->ev_pairs.resize(ev0);
    ctx->ev_recycle.resize(ev0);
    const int64_t nl = ctx->launches - l0;
    ctx->launches = l0;
    cudaGraphExec_t ex = nullptr;
    const bool good = s == DDKS_OK && e == cudaSuccess && g && ctx->alloc_epoch == key.epoch &&
                      cudaGraphInstantiate(&ex, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    if (!good) {
        cudaGetLastError();
        for (auto& v : evs) ctx->ev_free.push_back(v);
        ctx->err.clear();
        return DDKS_OK;
    }
    ctx->sg_exec = ex;
    ctx->sg_key = key;
    ctx->sg_launches = nl;
    ctx->sg_kd_levels = ctx->kd_levels;
    ctx->sg_rank_lanes = ctx->rank_lanes;
    ctx->sg_evs = evs;
    ctx->sg_ev_pairs = pairs;
    *ok = true;
    return DDKS_OK;
}





// a1-a7 for one pair, origins sharded across ranks; optional per-origin export (debug path, single rank).
// shard_world > 0: compute only the origin shard that rank shard_rank of shard_world would own (ddks_stat_shard).
// Repeated identical ddks_stat calls (same input pointers and sizes, same workspace) are captured into a CUDA graph
// on the second call and replayed with one cudaGraphLaunch from then on (DDKS_FLAG_NO_GRAPH disables it).
static ddks_status stat_impl(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int32_t d,
                             void* stream, ddks_result* out, int64_t o_begin_req, int64_t o_end_req,
                             uint64_t* per_origin_out, int shard_world = 0, int shard_rank = 0) {
    ctx->err.clear();
    ddks_status s = check_sizes(ctx, n_P, n_Q, d);
    if (s) return s;
    if (!P || !Q) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "null argument");
    s = bind_device(ctx);
    if (s) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t N = n_P + n_Q;
    const bool export_mode = per_origin_out != nullptr;
    int64_t ob, oe;
    if (export_mode) {
        ob = o_begin_req;
        oe = o_end_req;
    } else if (shard_world > 0) {
        ddks_shard_range(N, shard_world, shard_rank, &ob, &oe);
    } else {
        ddks_shard_range(N, ctx->world, ctx->rank, &ob, &oe);
    }
    const int sw = shard_world > 0 ? shard_world : ctx->world, sr = shard_world > 0 ? shard_rank : ctx->rank;
    if ((s = ensure_host(ctx, std::max<size_t>(4096, (size_t)ctx->world * sizeof(DevResult))))) return s;
    // the fused small-N path (whole statistic, single rank): one record per origin block
    const bool small = !export_mode && shard_world == 0 && small_fused_applies(ctx, n_P, n_Q);
    // environment overrides (tuning / test knobs) change the plan: a graph captured under other values is not reused
    const bool env_override = env_overrides();
    const bool graphable = !export_mode && shard_world == 0 && !(ctx->flags & DDKS_FLAG_NO_GRAPH) && !env_override &&
                           graph_input_ok(P) && graph_input_ok(Q);
    const ddks_ctx::StatKey key{P, Q, n_P, n_Q, d, ctx->alloc_epoch};
    bool replay = graphable && ctx->sg_exec && ctx->sg_key == key;
    if (graphable && !replay && ctx->sg_seen == key) {
        if ((s = stat_capture(ctx, key, P, n_P, Q, n_Q, d, ob, oe, sw, sr, &replay))) return s;
    }
    DevResult* hres;
    if (replay) {
        hres = (DevResult*)ctx->host_pinned;
        *hres = DevResult{0ull, ~0ull, 0ull, 0u, 0u};  // the graph's first node copies it to the device
        CU(cudaGraphLaunch(ctx->sg_exec, st));
        ctx->launches += ctx->sg_launches;
        ctx->kd_levels = ctx->sg_kd_levels;
        ctx->rank_lanes = ctx->sg_rank_lanes;
        for (size_t i = 0; i < ctx->sg_evs.size(); ++i) {
            ctx->ev_pending.push_back(ctx->sg_evs[i]);
            ctx->ev_pairs.push_back(ctx->sg_ev_pairs[i]);
            ctx->ev_recycle.push_back(0);
        }
    } else {
        if ((s = stat_enqueue(ctx, P, n_P, Q, n_Q, d, st, ob, oe, per_origin_out, sw, sr, small))) return s;
        hres = (DevResult*)ctx->host_pinned;
        if (graphable) {  // a second identical call (same workspace) will be captured
            ctx->sg_seen = key;
            ctx->sg_seen.epoch = ctx->alloc_epoch;
        }
    }
    CU(cudaStreamSynchronize(st));
    if ((s = collect_profile(ctx))) return s;
    // this rank's record, or (world > 1) the all-gathered records of every rank, combined on the host; the fused
    // small-N path left one record per origin block {num, key, flags}
    const bool use_key = small || (!export_mode && argmax_key_fits(n_P, n_Q));
    const int nrec = small ? (int)small_blocks(n_P + n_Q) : ((ctx->comm && !export_mode) ? ctx->world : 1);
    ddks_rank_record recs[64], comb;
    std::vector<ddks_rank_record> big;
    ddks_rank_record* rp = recs;
    if (nrec > 64) {
        big.resize(nrec);
        rp = big.data();
    }
    for (int r = 0; r < nrec; ++r) {
        if (small) {
            const unsigned long long* sr = (const unsigned long long*)ctx->host_pinned + 4 * r;
            rp[r] = decode_record(DevResult{sr[0], ~0ull, sr[1], (uint32_t)sr[2], 0u}, n_P, n_Q, true);
        } else {
            rp[r] = decode_record(hres[r], n_P, n_Q, use_key);
        }
    }
    ddks_combine_records(rp, nrec, &comb);
    if (comb.flags & 1u) return fail(ctx, DDKS_ERR_NONFINITE, "non-finite coordinate in input");
    if (out) {
        out->num = comb.num;
        out->den = (uint64_t)n_P * (uint64_t)n_Q;
        out->D = (double)out->num / (double)out->den;
        out->argmax_origin = comb.argmax_origin;
    }
    return DDKS_OK;
}

ddks_status ddks_stat(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int32_t d,
                      void* stream, ddks_result* out) {
    if (!ctx) return DDKS_ERR_INVALID_ARGUMENT;
    if (!out) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "null out");
    return stat_impl(ctx, P, n_P, Q, n_Q, d, stream, out, 0, 0, nullptr);
}

ddks_status ddks_stat_shard(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int32_t d,
                            int world, int rank, void* stream, ddks_result* out) {
    if (!ctx) return DDKS_ERR_INVALID_ARGUMENT;
    if (!out) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "null out");
    if (ctx->world != 1) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "ddks_stat_shard needs a single-rank context");
    if (world < 1 || rank < 0 || rank >= world) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "bad world/rank");
    return stat_impl(ctx, P, n_P, Q, n_Q, d, stream, out, 0, 0, nullptr, world, rank);
}

ddks_status ddks_stat_per_origin(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int32_t d,
                                 int64_t o_begin, int64_t o_end, uint64_t* num_out, void* stream) {
    if (!ctx) return DDKS_ERR_INVALID_ARGUMENT;
    if (!num_out) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "null num_out");
    if (o_begin < 0 || o_end < o_begin || o_end > n_P + n_Q)
        return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "bad origin range [%lld, %lld)", (long long)o_begin, (long long)o_end);
    if (o_end == o_begin) {
        ddks_status s = check_sizes(ctx, n_P, n_Q, d);
        return s;
    }
    return stat_impl(ctx, P, n_P, Q, n_Q, d, stream, nullptr, o_begin, o_end, num_out);
}

// item chunks of a host-input batch whose H2D copies overlap the counts of the earlier chunks
static constexpr int kCopyChunks = 4;  // C4 e2e 2.73 -> 2.04 ms (8 chunks: 2.23)

ddks_status ddks_stat_batch(ddks_ctx* ctx, const float* P, const float* Q, int64_t B, int64_t n_P, int64_t n_Q,
                            int32_t d, void* stream, ddks_result* out) {
    if (!ctx) return DDKS_ERR_INVALID_ARGUMENT;
    ctx->err.clear();
    if (B < 1) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "B=%lld < 1", (long long)B);
    ddks_status s = check_sizes(ctx, n_P, n_Q, d);
    if (s) return s;
    if (!P || !Q || !out) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "null argument");
    if ((s = bind_device(ctx))) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t N = n_P + n_Q;
    const int DP = pad_dim(d);
    int64_t ib, ie;
    ddks_shard_range(B, ctx->world, ctx->rank, &ib, &ie);
    const int64_t gstride = ctx->comm ? gather_stride(B, ctx->world, 1) : 0;
    // host inputs (this rank's items >= 8 MB): H2D in chunks of items on the copy stream, each chunk's pack + count
    // waiting only for its own copy, so the transfer of chunk c + 1 overlaps the count of chunk c
    const int64_t nb_items = ie - ib;
    const size_t item_bytes = (size_t)(n_P + n_Q) * d * 4;
    const bool host_in = !is_device_ptr(P) && !is_device_ptr(Q);
    const int nchunk = (host_in && nb_items >= 2 && nb_items * item_bytes >= ((size_t)8 << 20))
                           ? (int)std::min<int64_t>(kCopyChunks, nb_items) : 1;
    auto enq = [&](cudaStream_t st) -> ddks_status {
        ddks_status s;
        const void *dP, *dQ;
        if (nchunk > 1) {
            if ((s = ensure(ctx, ctx->raw_a, (size_t)B * n_P * d * 4))) return s;
            if ((s = ensure(ctx, ctx->raw_b, (size_t)B * n_Q * d * 4))) return s;
            dP = ctx->raw_a.p;
            dQ = ctx->raw_b.p;
        } else {
            if ((s = stage_input(ctx, P, (size_t)B * n_P * d * 4, ctx->raw_a, st, &dP))) return s;
            if ((s = stage_input(ctx, Q, (size_t)B * n_Q * d * 4, ctx->raw_b, st, &dQ))) return s;
        }
        if ((s = ensure(ctx, ctx->item_num, (size_t)B * 8))) return s;
        uint64_t* nums = (uint64_t*)ctx->item_num.p;
        CU(cudaMemsetAsync(nums, 0, (size_t)B * 8, st));
        DevResult* dres = (DevResult*)ctx->res.p;
        CU(cudaMemsetAsync(dres, 0, sizeof(DevResult), st));
        const int64_t nb = ie - ib;
        if (nb > 0) {
            if ((s = ensure(ctx, ctx->packed, (size_t)nb * N * DP * 4))) return s;
            float* packed = (float*)ctx->packed.p;
            if (nchunk > 1) {  // fork the copy stream off st (so a capture follows it), queue every chunk's copies
                if (!ctx->copy_stream) CU(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
                while ((int)ctx->copy_evs.size() < nchunk + 1) {
                    cudaEvent_t e;
                    CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
                    ctx->copy_evs.push_back(e);
                }
                CU(cudaEventRecord(ctx->copy_evs[nchunk], st));
                CU(cudaStreamWaitEvent(ctx->copy_stream, ctx->copy_evs[nchunk], 0));
                for (int c = 0; c < nchunk; ++c) {
                    const int64_t c0 = ib + nb * c / nchunk, c1 = ib + nb * (c + 1) / nchunk;
                    CU(cudaMemcpyAsync((float*)ctx->raw_a.p + c0 * n_P * d, P + c0 * n_P * d,
                                       (size_t)(c1 - c0) * n_P * d * 4, cudaMemcpyHostToDevice, ctx->copy_stream));
                    CU(cudaMemcpyAsync((float*)ctx->raw_b.p + c0 * n_Q * d, Q + c0 * n_Q * d,
                                       (size_t)(c1 - c0) * n_Q * d * 4, cudaMemcpyHostToDevice, ctx->copy_stream));
                    CU(cudaEventRecord(ctx->copy_evs[c], ctx->copy_stream));
                }
            }
            for (int c = 0; c < nchunk; ++c) {  // chunk c: items [c0, c1) of this rank's [ib, ie)
                const int64_t c0 = ib + nb * c / nchunk, c1 = ib + nb * (c + 1) / nchunk;
                if (nchunk > 1) CU(cudaStreamWaitEvent(st, ctx->copy_evs[c], 0));  // (joins the copy stream at the end)
                bool wx = false;
                float* pk = packed + (c0 - ib) * N * DP;
                if ((s = launch_pack_batch(ctx, (const float*)dP + c0 * n_P * d, n_P, (const float*)dQ + c0 * n_Q * d,
                                           n_Q, d, c1 - c0, pk, &dres->flag, st, &wx)))
                    return s;
                if ((s = run_count(ctx, pk, d, c1 - c0, n_P, n_Q, 0, N, nums + c0, nullptr, st, false, nullptr, wx)))
                    return s;
            }
        }
        // world > 1: one all-gather of the padded per-rank records (this rank's nums + its flags), unpadded on the
        // host
        if ((s = ensure_host(ctx, sizeof(DevResult) + (size_t)B * 8 + (size_t)ctx->world * gstride * 8))) return s;
        DevResult* hres = (DevResult*)ctx->host_pinned;
        uint64_t* hnums = (uint64_t*)((char*)ctx->host_pinned + sizeof(DevResult));
        if (ctx->comm) {
            uint64_t* arrs[1] = {nums};
            if ((s = gather_items(ctx, arrs, 1, B, &dres->flag, st, hnums + B))) return s;
        } else {
            CU(cudaMemcpyAsync(hres, dres, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
            CU(cudaMemcpyAsync(hnums, nums, (size_t)B * 8, cudaMemcpyDeviceToHost, st));
        }
        return DDKS_OK;
    };
    const std::vector<uint64_t> key{(uint64_t)(uintptr_t)P, (uint64_t)(uintptr_t)Q, (uint64_t)B, (uint64_t)n_P,
                                    (uint64_t)n_Q, (uint64_t)d, (uint64_t)ctx->flags};
    if ((s = run_call(ctx, ctx->cg_batch, key, graph_input_ok(P) && graph_input_ok(Q), st, enq))) return s;
    CU(cudaStreamSynchronize(st));
    DevResult* hres = (DevResult*)ctx->host_pinned;
    uint64_t* hnums = (uint64_t*)((char*)ctx->host_pinned + sizeof(DevResult));
    uint64_t* hgath = hnums + B;
    if ((s = collect_profile(ctx))) return s;
    if (ctx->comm) ddks_unpad_items(hgath, B, ctx->world, 1, hnums, &hres->flag);
    if (hres->flag & 1u) return fail(ctx, DDKS_ERR_NONFINITE, "non-finite coordinate in input");
    const uint64_t den = (uint64_t)n_P * (uint64_t)n_Q;
    for (int64_t b = 0; b < B; ++b) {
        out[b].num = hnums[b];
        out[b].den = den;
        out[b].D = (double)hnums[b] / (double)den;
        out[b].argmax_origin = -1;
    }
    return DDKS_OK;
}

ddks_status ddks_permutation_null(ddks_ctx* ctx, const float* pooled, int64_t n_P, int64_t n_Q, int32_t d,
                                  const int32_t* perms, int64_t n_perm, void* stream, uint64_t* null_num,
                                  ddks_result* observed, double* p_value) {
    if (!ctx) return DDKS_ERR_INVALID_ARGUMENT;
    ctx->err.clear();
    if (n_perm < 0) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "n_perm < 0");
    ddks_status s = check_sizes(ctx, n_P, n_Q, d);
    if (s) return s;
    if (!pooled || (n_perm > 0 && !perms)) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "null argument");
    if ((s = bind_device(ctx))) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t N = n_P + n_Q;
    // slot 0 = observed (identity split), slots 1..n_perm = permutations
    const int64_t total = n_perm + 1;
    const int64_t gstride = ctx->comm ? gather_stride(n_perm, ctx->world, 1) : 0;
    const bool obs_small = small_fused_applies(ctx, n_P, n_Q);
    const int64_t nsrec = obs_small ? small_blocks(N) : 0;
    const int DP = pad_dim(d);
    auto enq = [&](cudaStream_t st) -> ddks_status {
        ddks_status s;
        const void *dpool, *dperm = nullptr;
        if ((s = stage_input(ctx, pooled, (size_t)N * d * 4, ctx->raw_a, st, &dpool))) return s;
        if (n_perm > 0 && (s = stage_input(ctx, perms, (size_t)n_perm * N * 4, ctx->raw_perm, st, &dperm))) return s;
        if ((s = ensure(ctx, ctx->item_num, (size_t)total * 8))) return s;
        uint64_t* nums = (uint64_t*)ctx->item_num.p;
        CU(cudaMemsetAsync(nums, 0, (size_t)total * 8, st));
        DevResult* dres = (DevResult*)ctx->res.p;
        CU(cudaMemsetAsync(dres, 0, sizeof(DevResult), st));
        // pack the pooled sample once: [N][DP], rows up to a multiple of the tensor-core null's k-block zeroed
        const int64_t N_pad = (N + ddks::PM_KB - 1) / ddks::PM_KB * ddks::PM_KB;
        if ((s = ensure(ctx, ctx->pool_packed, (size_t)N_pad * DP * 4))) return s;
        float* pooled_packed = (float*)ctx->pool_packed.p;
        if (N_pad > N) CU(cudaMemsetAsync(pooled_packed + N * DP, 0, (size_t)(N_pad - N) * DP * 4, st));
        if ((s = launch_pack(ctx, (const float*)dpool, n_P, (const float*)dpool + n_P * d, n_Q, d, 1, pooled_packed,
                             &dres->flag, st)))
            return s;
        // pinned host layout: result record, total nums, the all-gathered rank records (world > 1), and the fused small
        // statistic's per-origin-block records (allocated before anything is enqueued: the small kernel writes there)
        if ((s = ensure_host(ctx, sizeof(DevResult) + (size_t)(total + (size_t)ctx->world * gstride + 4 * nsrec) * 8)))
            return s;
        unsigned long long* hsrec =
            (unsigned long long*)((char*)ctx->host_pinned + sizeof(DevResult)) + total + (size_t)ctx->world * gstride;
        // observed: every rank computes it (cheap relative to the null), no collective needed; at small N (single rank)
        // the fused cluster kernel on the raw halves of the pooled sample (its records land in hsrec, combined below)
        if (obs_small) {
            if ((s = small_enqueue(ctx, (const float*)dpool, n_P, (const float*)dpool + n_P * d, n_Q, d, st, hsrec))) return s;
        } else if ((s = run_count(ctx, pooled_packed, d, 1, n_P, n_Q, 0, N, nums, nullptr, st))) {
            return s;
        }
        int64_t jb, je;
        ddks_shard_range(n_perm, ctx->world, ctx->rank, &jb, &je);
        const bool label_path = N <= 65535 && !(ctx->flags & DDKS_FLAG_PERM_GATHER);
        if (label_path) {
            auto fn = perm_mma_applies(ctx, d, N) ? launch_perm_mma : launch_perm;
            // permutations in groups whose label images / counters and validation bitmaps stay within ~256 MB (about
            // 1.5 N bytes per permutation; DDKS_PERM_GROUP, test only, overrides the group size)
            int64_t grp = std::max<int64_t>(768, ((256ll << 20) / (3 * N / 2 + 1)) / 768 * 768);
            if (const char* e = getenv("DDKS_PERM_GROUP")) grp = std::max(1, atoi(e));
            for (int64_t j0 = jb; j0 < je; j0 += grp) {
                const int64_t nj = std::min(grp, je - j0);
                if ((s = fn(ctx, d, pooled_packed, (const int32_t*)dperm + j0 * N, nj, n_P, n_Q, nums + 1 + j0, &dres->flag,
                            st)))
                    return s;
            }
        } else {
            const int64_t chunk_max = std::max<int64_t>(1, (int64_t)((256ull << 20) / ((size_t)N * DP * 4)));
            for (int64_t j0 = jb; j0 < je; j0 += chunk_max) {
                const int64_t nc = std::min(chunk_max, je - j0);
                if ((s = ensure(ctx, ctx->packed, (size_t)nc * N * DP * 4))) return s;
                const int64_t words = (N + 31) / 32;
                if ((s = ensure(ctx, ctx->bitmap, (size_t)nc * words * 4))) return s;
                CU(cudaMemsetAsync(ctx->bitmap.p, 0, (size_t)nc * words * 4, st));
                const int64_t tot = nc * N;
                const int blocks = (int)std::min<int64_t>((tot + 255) / 256, 148 * 8);
                if (DP == 4)
                    ddks::k_gather<4><<<blocks, 256, 0, st>>>(pooled_packed, (const int32_t*)dperm + j0 * N, nc, N,
                                                              (float*)ctx->packed.p, (uint32_t*)ctx->bitmap.p, &dres->flag);
                else
                    ddks::k_gather<8><<<blocks, 256, 0, st>>>(pooled_packed, (const int32_t*)dperm + j0 * N, nc, N,
                                                              (float*)ctx->packed.p, (uint32_t*)ctx->bitmap.p, &dres->flag);
                CHECK_LAUNCH();
                ctx->launches++;
                if ((s = run_count(ctx, (const float*)ctx->packed.p, d, nc, n_P, n_Q, 0, N, nums + 1 + j0, nullptr, st)))
                    return s;
            }
        }
        // world > 1: the observed num (slot 0) is every rank's own; one all-gather of the padded per-rank records (this
        // rank's permutation nums + its flags), unpadded on the host
        DevResult* hres = (DevResult*)ctx->host_pinned;
        uint64_t* hnums = (uint64_t*)((char*)ctx->host_pinned + sizeof(DevResult));
        uint64_t* hgath = hnums + total;
        if (ctx->comm) {
            uint64_t* arrs[1] = {nums + 1};
            if ((s = gather_items(ctx, arrs, 1, n_perm, &dres->flag, st, hgath))) return s;
            CU(cudaMemcpyAsync(hnums, nums, 8, cudaMemcpyDeviceToHost, st));
        } else {
            CU(cudaMemcpyAsync(hres, dres, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
            CU(cudaMemcpyAsync(hnums, nums, (size_t)total * 8, cudaMemcpyDeviceToHost, st));
        }
        return DDKS_OK;
    };
    const std::vector<uint64_t> key{(uint64_t)(uintptr_t)pooled, (uint64_t)(uintptr_t)perms, (uint64_t)n_P,
                                    (uint64_t)n_Q, (uint64_t)d, (uint64_t)n_perm, (uint64_t)ctx->flags};
    if ((s = run_call(ctx, ctx->cg_null, key, graph_input_ok(pooled) && (n_perm == 0 || graph_input_ok(perms)), st,
                      enq)))
        return s;
    DevResult* hres = (DevResult*)ctx->host_pinned;
    uint64_t* hnums = (uint64_t*)((char*)ctx->host_pinned + sizeof(DevResult));
    uint64_t* hgath = hnums + total;
    const unsigned long long* hsrec = (const unsigned long long*)hgath + (size_t)ctx->world * gstride;
    CU(cudaStreamSynchronize(st));
    if ((s = collect_profile(ctx))) return s;
    if (ctx->comm) ddks_unpad_items(hgath, n_perm, ctx->world, 1, hnums + 1, &hres->flag);
    if (hres->flag & 1u) return fail(ctx, DDKS_ERR_NONFINITE, "non-finite coordinate in input");
    if (hres->flag & 2u) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "a perms row is not a permutation of 0..N-1");
    if (obs_small) {  // the fused statistic's per-origin-block records {num, key, flags}
        std::vector<ddks_rank_record> recs((size_t)nsrec);
        for (int64_t r = 0; r < nsrec; ++r) {
            const unsigned long long* sr = hsrec + 4 * r;
            recs[r] = decode_record(DevResult{sr[0], ~0ull, sr[1], (uint32_t)sr[2], 0u}, n_P, n_Q, true);
        }
        ddks_rank_record comb;
        ddks_combine_records(recs.data(), (int)nsrec, &comb);
        if (comb.flags & 1u) return fail(ctx, DDKS_ERR_NONFINITE, "non-finite coordinate in input");
        hnums[0] = comb.num;
    }
    const uint64_t obs = hnums[0];
    int64_t ge = 0;
    for (int64_t j = 0; j < n_perm; ++j) {
        if (null_num) null_num[j] = hnums[1 + j];
        if (hnums[1 + j] >= obs) ++ge;
    }
    if (observed) {
        observed->num = obs;
        observed->den = (uint64_t)n_P * (uint64_t)n_Q;
        observed->D = (double)obs / (double)observed->den;
        observed->argmax_origin = -1;
    }
    if (p_value) *p_value = (double)(1 + ge) / (double)(1 + n_perm);
    return DDKS_OK;
}

}  // extern "C"
