// ddks_api_significance.cu — C-ABI entry ddks_significance (include/ddks.h; §3).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "ddks_internal.h"
#include "ddks_significance.cuh"

using namespace ddks_host;

extern "C" {

// ------------------------------------------------------------------------------------- analytic significance
// PAPER.md §3, SURVEY §8f NEXT-1. One SPLIT classify+count pass gives num (as ddks_stat) and the
// histogram of the Q-counts M_T over the 2^d x N cells; the per-cell factor log p(d <= D | lambda) depends only on
// M_T, so it is tabulated for the distinct values (k_sig_table) and summed with the histogram as weights.
ddks_status ddks_significance(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int32_t d,
                              uint32_t sig_flags, void* stream, ddks_significance_result* out, uint64_t* mt_hist,
                              double* log_p_table) {
    if (!ctx) return DDKS_ERR_INVALID_ARGUMENT;
    ctx->err.clear();
    if (!out) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "null out");
    if (sig_flags & ~DDKS_SIG_POISSON) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "bad sig_flags");
    ddks_status s = check_sizes(ctx, n_P, n_Q, d);
    if (s) return s;
    if (!P || !Q) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "null argument");
    if ((s = bind_device(ctx))) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t N = n_P + n_Q;
    const int DP = pad_dim(d);
    int64_t ob, oe;
    ddks_shard_range(N, ctx->world, ctx->rank, &ob, &oe);
    const void *dP, *dQ;
    if ((s = stage_input(ctx, P, (size_t)n_P * d * 4, ctx->raw_a, st, &dP))) return s;
    if ((s = stage_input(ctx, Q, (size_t)n_Q * d * 4, ctx->raw_b, st, &dQ))) return s;
    if ((s = ensure(ctx, ctx->packed, (size_t)N * DP * 4))) return s;
    const int64_t nm = n_Q + 1;  // M_T in 0..n_Q
    const int64_t n_max = std::max(n_P, n_Q);
    // log n! for n <= n_max, plus room for the Poisson mass beyond N (mean < N, ~14 sd above it is below e^-100)
    const int64_t n_lf = n_max + 1 + ((sig_flags & DDKS_SIG_POISSON) ? (int64_t)(32.0 * std::sqrt((double)n_max)) + 2048 : 0);
    if ((s = ensure(ctx, ctx->sig_hist, (size_t)nm * 8))) return s;
    if ((s = ensure(ctx, ctx->sig_lf, (size_t)n_lf * 8))) return s;
    if ((s = ensure(ctx, ctx->sig_table, (size_t)nm * 8))) return s;
    if ((s = ensure(ctx, ctx->sig_contrib, (size_t)nm * 8))) return s;
    if ((s = ensure(ctx, ctx->sig_part, (size_t)ctx->world * 8 + 8))) return s;
    unsigned long long* hist = (unsigned long long*)ctx->sig_hist.p;
    double* LF = (double*)ctx->sig_lf.p;
    double* table = (double*)ctx->sig_table.p;
    double* contrib = (double*)ctx->sig_contrib.p;
    double* part = (double*)ctx->sig_part.p;  // [0] = this rank's partial sum, [1 + r] = gathered partials
    CU(cudaMemsetAsync(hist, 0, (size_t)nm * 8, st));
    CU(cudaMemsetAsync(table, 0, (size_t)nm * 8, st));
    CU(cudaMemsetAsync(contrib, 0, (size_t)nm * 8, st));
    DevResult* dres = (DevResult*)ctx->res.p;
    DevResult* hres = (DevResult*)ctx->host_pinned;
    *hres = DevResult{0ull, ~0ull, 0ull, 0u, 0u};
    CU(cudaMemcpyAsync(dres, hres, sizeof(DevResult), cudaMemcpyHostToDevice, st));
    float* packed = (float*)ctx->packed.p;
    if ((s = launch_pack(ctx, (const float*)dP, n_P, (const float*)dQ, n_Q, d, 1, packed, &dres->flag, st))) return s;
    uint64_t* per = nullptr;
    if ((s = count_statistic(ctx, packed, d, n_P, n_Q, ob, oe, ctx->world, ctx->rank, dres, false, true, hist, st, &per,
                             true)))
        return s;
    const bool use_key = argmax_key_fits(n_P, n_Q);
    if (ctx->comm) {
        if (use_key) {  // (the k_argmax path all-reduced num inside count_statistic)
            NC(ncclAllReduce(&dres->num, &dres->num, 1, ncclUint64, ncclMax, ctx->comm, st));
            NC(ncclAllReduce(&dres->key, &dres->key, 1, ncclUint64, ncclMax, ctx->comm, st));
        }
        NC(ncclAllReduce(&dres->arg, &dres->arg, 1, ncclUint64, ncclMin, ctx->comm, st));
        NC(ncclAllReduce(&dres->flag, &dres->flag, 1, ncclUint32, ncclMax, ctx->comm, st));
        NC(ncclAllReduce(hist, hist, (size_t)nm, ncclUint64, ncclSum, ctx->comm, st));
    }
    ddks::k_logfact<<<(int)std::min<int64_t>((n_lf + 255) / 256, 148 * 8), 256, 0, st>>>(LF, n_lf - 1);
    CHECK_LAUNCH();
    ctx->launches++;
    // table entries [mb, me) on this rank
    int64_t mb, me;
    ddks_shard_range(nm, ctx->world, ctx->rank, &mb, &me);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(me - mb, 148 * 2));
    // window bound: ~2 x sqrt(2 x 100) standard deviations (+ slack for skewed small-rate pmfs); a kernel that
    // finds a wider window flags it and the table is recomputed with twice the scratch
    const double var = (sig_flags & DDKS_SIG_POISSON) ? (double)n_max : (double)n_max / 4.0;
    int64_t W_max = std::min<int64_t>(n_max + 1, (int64_t)(32.0 * std::sqrt(var)) + 512);
    const uint64_t host_part_off = sizeof(DevResult);
    if ((s = ensure_host(ctx, host_part_off + (size_t)(ctx->world + 1) * 8))) return s;
    hres = (DevResult*)ctx->host_pinned;
    double* hpart = (double*)((char*)ctx->host_pinned + host_part_off);
    for (int attempt = 0;; ++attempt) {
        if ((s = ensure(ctx, ctx->sig_scratch, (size_t)grid * 2 * W_max * 8))) return s;
        ddks::SigArgs sa{};
        sa.LF = LF;
        sa.lf_max = n_lf - 1;
        sa.hist = hist;
        sa.num = (const unsigned long long*)&dres->num;
        sa.N_P = n_P;
        sa.N_T = n_Q;
        sa.m_begin = mb;
        sa.m_end = me;
        sa.poisson = (sig_flags & DDKS_SIG_POISSON) ? 1 : 0;
        sa.scratch = (double*)ctx->sig_scratch.p;
        sa.W_max = W_max;
        sa.table = table;
        sa.contrib = contrib;
        sa.flag = &dres->flag;
        if (me > mb) {
            ddks::k_sig_table<<<grid, ddks::SIG_T, 0, st>>>(sa);
            CHECK_LAUNCH();
            ctx->launches++;
        }
        ddks::k_sig_sum<<<1, ddks::SIG_T, 0, st>>>(contrib, mb, me, part);
        CHECK_LAUNCH();
        ctx->launches++;
        if (ctx->comm) {
            NC(ncclAllReduce(&dres->flag, &dres->flag, 1, ncclUint32, ncclMax, ctx->comm, st));
            NC(ncclAllGather(part, part + 1, 1, ncclFloat64, ctx->comm, st));
        } else {
            CU(cudaMemcpyAsync(part + 1, part, 8, cudaMemcpyDeviceToDevice, st));
        }
        CU(cudaMemcpyAsync(hres, dres, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(hpart, part + 1, (size_t)ctx->world * 8, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        if ((s = collect_profile(ctx))) return s;
        if (hres->flag & 1u) return fail(ctx, DDKS_ERR_NONFINITE, "non-finite coordinate in input");
        if (!(hres->flag & 4u)) break;
        if (attempt >= 3 || W_max >= n_max + 1) return fail(ctx, DDKS_ERR_CUDA, "significance window exceeds scratch");
        W_max = std::min<int64_t>(n_max + 1, 2 * W_max);
        const uint32_t zero = 0;
        CU(cudaMemcpyAsync(&dres->flag, &zero, 4, cudaMemcpyHostToDevice, st));
    }
    double log_prod = 0.0;
    for (int r = 0; r < ctx->world; ++r) log_prod += hpart[r];  // rank order: deterministic
    if (mt_hist) {
        CU(cudaMemcpyAsync(mt_hist, hist, (size_t)nm * 8, cudaMemcpyDefault, st));
    }
    if (log_p_table) {
        if (ctx->comm) NC(ncclAllReduce(table, table, (size_t)nm, ncclFloat64, ncclSum, ctx->comm, st));
        CU(cudaMemcpyAsync(log_p_table, table, (size_t)nm * 8, cudaMemcpyDefault, st));
    }
    CU(cudaStreamSynchronize(st));
    const ddks_rank_record rec = decode_record(*hres, n_P, n_Q, use_key);
    out->stat.num = rec.num;
    out->stat.den = (uint64_t)n_P * (uint64_t)n_Q;
    out->stat.D = (double)out->stat.num / (double)out->stat.den;
    out->stat.argmax_origin = rec.argmax_origin;
    out->log_prod = log_prod;
    out->S = 0.0 - std::expm1(log_prod);  // (0.0 - x: no negative zero when log_prod == 0)
    out->cells = ((int64_t)1 << d) * N;
    return DDKS_OK;
}

// ------------------------------------------------------------------------------------- batched significance
// B independent pairs (the paper's power analyses repeat small tests): one SPLIT count
// launch for all items (per-item M_T histograms), one table launch over all (item, m) entries, one sum per item.
// Items are sharded across ranks; every rank returns all B results (all-gather of num and log_prod).
ddks_status ddks_significance_batch(ddks_ctx* ctx, const float* P, const float* Q, int64_t B, int64_t n_P,
                                    int64_t n_Q, int32_t d, uint32_t sig_flags, void* stream,
                                    ddks_significance_result* out) {
    if (!ctx) return DDKS_ERR_INVALID_ARGUMENT;
    ctx->err.clear();
    if (!out || !P || !Q) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "null argument");
    if (B < 1) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "B=%lld < 1", (long long)B);
    if (sig_flags & ~DDKS_SIG_POISSON) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "bad sig_flags");
    ddks_status s = check_sizes(ctx, n_P, n_Q, d);
    if (s) return s;
    if ((s = bind_device(ctx))) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t N = n_P + n_Q;
    const int DP = pad_dim(d);
    const int64_t nm = n_Q + 1;
    int64_t ib, ie;
    ddks_shard_range(B, ctx->world, ctx->rank, &ib, &ie);
    const int64_t nb = ie - ib;
    const void *dP, *dQ;
    if ((s = stage_input(ctx, P, (size_t)B * n_P * d * 4, ctx->raw_a, st, &dP))) return s;
    if ((s = stage_input(ctx, Q, (size_t)B * n_Q * d * 4, ctx->raw_b, st, &dQ))) return s;
    const int64_t n_max = std::max(n_P, n_Q);
    const int64_t n_lf = n_max + 1 + ((sig_flags & DDKS_SIG_POISSON) ? (int64_t)(32.0 * std::sqrt((double)n_max)) + 2048 : 0);
    const size_t cells = (size_t)std::max<int64_t>(nb, 1) * nm;
    if ((s = ensure(ctx, ctx->sig_hist, cells * 8))) return s;
    if ((s = ensure(ctx, ctx->sig_lf, (size_t)n_lf * 8))) return s;
    if ((s = ensure(ctx, ctx->sig_table, cells * 8))) return s;
    if ((s = ensure(ctx, ctx->sig_contrib, cells * 8))) return s;
    if ((s = ensure(ctx, ctx->item_num, (size_t)B * 8))) return s;
    if ((s = ensure(ctx, ctx->sig_part, (size_t)B * 8))) return s;
    unsigned long long* hist = (unsigned long long*)ctx->sig_hist.p;
    double* LF = (double*)ctx->sig_lf.p;
    double* table = (double*)ctx->sig_table.p;
    double* contrib = (double*)ctx->sig_contrib.p;
    uint64_t* nums = (uint64_t*)ctx->item_num.p;
    double* parts = (double*)ctx->sig_part.p;
    CU(cudaMemsetAsync(hist, 0, cells * 8, st));
    CU(cudaMemsetAsync(nums, 0, (size_t)B * 8, st));
    CU(cudaMemsetAsync(parts, 0, (size_t)B * 8, st));
    DevResult* dres = (DevResult*)ctx->res.p;
    CU(cudaMemsetAsync(dres, 0, sizeof(DevResult), st));
    if (nb > 0) {
        if ((s = ensure(ctx, ctx->packed, (size_t)nb * N * DP * 4))) return s;
        float* packed = (float*)ctx->packed.p;
        bool wx = false;  // small items: near-x_0-sorted runs, warp-level bit 0 (the M_T histogram is order-free)
        if ((s = launch_pack_batch(ctx, (const float*)dP + ib * n_P * d, n_P, (const float*)dQ + ib * n_Q * d, n_Q, d,
                                   nb, packed, &dres->flag, st, &wx)))
            return s;
        if ((s = run_count(ctx, packed, d, nb, n_P, n_Q, 0, N, nums + ib, nullptr, st, true, hist, wx))) return s;
        ddks::k_logfact<<<(int)std::min<int64_t>((n_lf + 255) / 256, 148 * 8), 256, 0, st>>>(LF, n_lf - 1);
        CHECK_LAUNCH();
        ctx->launches++;
        const int64_t entries = nb * nm;
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(entries, 148 * 2));
        const double var = (sig_flags & DDKS_SIG_POISSON) ? (double)n_max : (double)n_max / 4.0;
        int64_t W_max = std::min<int64_t>(n_max + 1, (int64_t)(32.0 * std::sqrt(var)) + 512);
        for (int attempt = 0;; ++attempt) {
            if ((s = ensure(ctx, ctx->sig_scratch, (size_t)grid * 2 * W_max * 8))) return s;
            ddks::SigArgs sa{};
            sa.LF = LF;
            sa.lf_max = n_lf - 1;
            sa.hist = hist;
            sa.num = (const unsigned long long*)(nums + ib);
            sa.N_P = n_P;
            sa.N_T = n_Q;
            sa.m_begin = 0;
            sa.m_end = entries;
            sa.poisson = (sig_flags & DDKS_SIG_POISSON) ? 1 : 0;
            sa.scratch = (double*)ctx->sig_scratch.p;
            sa.W_max = W_max;
            sa.table = table;
            sa.contrib = contrib;
            sa.flag = &dres->flag;
            ddks::k_sig_table<<<grid, ddks::SIG_T, 0, st>>>(sa);
            ddks::k_sig_sum<<<(unsigned)nb, ddks::SIG_T, 0, st>>>(contrib, 0, nm, parts + ib, nm);
            CHECK_LAUNCH();
            ctx->launches += 2;
            uint32_t hflag = 0;
            CU(cudaMemcpyAsync(&hflag, &dres->flag, 4, cudaMemcpyDeviceToHost, st));
            CU(cudaStreamSynchronize(st));
            if (!(hflag & 4u)) break;
            if (attempt >= 3 || W_max >= n_max + 1) return fail(ctx, DDKS_ERR_CUDA, "significance window exceeds scratch");
            W_max = std::min<int64_t>(n_max + 1, 2 * W_max);
            CU(cudaMemsetAsync(&dres->flag, 0, 4, st));
        }
    }
    // world > 1: one all-gather of the padded per-rank records (nums, log_prod bits, flags), unpadded on the host
    const int64_t gstride = ctx->comm ? gather_stride(B, ctx->world, 2) : 0;
    if ((s = ensure_host(ctx, sizeof(DevResult) + (size_t)B * 16 + (size_t)ctx->world * gstride * 8))) return s;
    DevResult* hres = (DevResult*)ctx->host_pinned;
    uint64_t* hnums = (uint64_t*)((char*)ctx->host_pinned + sizeof(DevResult));
    double* hparts = (double*)(hnums + B);
    uint64_t* hgath = hnums + 2 * B;
    if (ctx->comm) {
        uint64_t* arrs[2] = {nums, (uint64_t*)parts};
        if ((s = gather_items(ctx, arrs, 2, B, &dres->flag, st, hgath))) return s;
    } else {
        CU(cudaMemcpyAsync(hres, dres, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(hnums, nums, (size_t)B * 8, cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(hparts, parts, (size_t)B * 8, cudaMemcpyDeviceToHost, st));
    }
    CU(cudaStreamSynchronize(st));
    if ((s = collect_profile(ctx))) return s;
    if (ctx->comm) ddks_unpad_items(hgath, B, ctx->world, 2, hnums, &hres->flag);  // nums then parts: contiguous
    if (hres->flag & 1u) return fail(ctx, DDKS_ERR_NONFINITE, "non-finite coordinate in input");
    const uint64_t den = (uint64_t)n_P * (uint64_t)n_Q;
    for (int64_t b = 0; b < B; ++b) {
        out[b].stat.num = hnums[b];
        out[b].stat.den = den;
        out[b].stat.D = (double)hnums[b] / (double)den;
        out[b].stat.argmax_origin = -1;
        out[b].log_prod = hparts[b];
        out[b].S = 0.0 - std::expm1(hparts[b]);
        out[b].cells = ((int64_t)1 << d) * N;
    }
    return DDKS_OK;
}

}  // extern "C"
