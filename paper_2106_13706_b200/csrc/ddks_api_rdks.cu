// ddks_api_rdks.cu — C-ABI entry ddks_rdks (include/ddks.h; §2.2.3, Alg. 2).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "ddks_internal.h"
#include "ddks_minmax.cuh"
#include "ddks_rdks.cuh"

using namespace ddks_host;

// about N / 4 distance buckets per corner, N / 8 from 2^20 rows (C5: 189 -> 175 us per graphed call; N / 8 is 2-3 us
// slower at C2 / C3, N / 16 slower everywhere: profiles/r2b_rdks_buckets.txt); DDKS_RDB_DIV (experiments) forces one
#ifndef DDKS_RDB_DIV
#define DDKS_RDB_DIV 0
#endif
static int64_t rdb_bucket_div(int64_t N) { return DDKS_RDB_DIV ? DDKS_RDB_DIV : (N >= (int64_t(1) << 20) ? 8 : 4); }

// distance keys (+ bucket counts when cnt): per point for d <= 8 (x' computed once), per (point, corner) otherwise
static void launch_rd_keys(const float* P, const float* Q, const double* xn, int64_t N, int64_t n_P, int d,
                           const uint32_t* keys, int cb, int ce, uint64_t* key, uint32_t* cnt, int nbk, double scale,
                           cudaStream_t st) {
    auto grid_for = [](int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); };
    switch (xn ? 0 : d) {
#define RDK(D) case D: ddks::k_rd_keys_pt<D><<<grid_for(N), 256, 0, st>>>(P, Q, N, n_P, keys, cb, ce, key, cnt, nbk, scale); return;
        RDK(1) RDK(2) RDK(3) RDK(4) RDK(5) RDK(6) RDK(7) RDK(8)
#undef RDK
        default:
            ddks::k_rd_keys<<<grid_for(N * (ce - cb)), 256, 0, st>>>(P, Q, xn, N, n_P, d, keys, cb, ce, key, cnt, nbk,
                                                                      scale);
    }
}

extern "C" {

// ------------------------------------------------------------------------------------- rdKS (Alg. 2)
// Corners sharded across ranks; the statistic is the max over corners (NCCL all-reduce max, then min of the first
// attaining corner index).
ddks_status ddks_rdks(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int32_t d,
                      void* stream, ddks_result* out) {
    if (!ctx) return DDKS_ERR_INVALID_ARGUMENT;
    ctx->err.clear();
    if (!out) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "null out");
    if (n_P < 0 || n_Q < 0) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "negative sample size");
    if (n_P == 0 || n_Q == 0) return fail(ctx, DDKS_ERR_EMPTY_SAMPLE, "empty sample");
    if (d < 1) return fail(ctx, DDKS_ERR_DIM_UNSUPPORTED, "d=%d < 1", d);
    const int64_t N = n_P + n_Q;
    if (N >= (int64_t(1) << 31) || (double)n_P * (double)n_Q >= 9007199254740992.0 ||
        (double)N * (double)(d + 1) >= (double)(int64_t(1) << 34))
        return fail(ctx, DDKS_ERR_TOO_LARGE, "rdKS problem too large (N=%lld, d=%d)", (long long)N, d);
    if (!P || !Q) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "null argument");
    ddks_status s;
    if ((s = bind_device(ctx))) return s;
    cudaStream_t st = (cudaStream_t)stream;
    int64_t cb, ce;
    ddks_shard_range(d + 1, ctx->world, ctx->rank, &cb, &ce);
    const int nc = (int)(ce - cb);
    const int tiles = (int)((N + ddks::RS_TILE - 1) / ddks::RS_TILE);
    if ((s = ensure(ctx, ctx->rd_keys, (size_t)2 * d * 4))) return s;
    if ((s = ensure(ctx, ctx->rd_k0, (size_t)std::max(nc, 1) * N * 8))) return s;
    if ((s = ensure(ctx, ctx->rd_k1, (size_t)std::max(nc, 1) * N * 8))) return s;
    if ((s = ensure(ctx, ctx->rd_hist, (size_t)std::max(nc, 1) * tiles * 256 * 4))) return s;
    if ((s = ensure(ctx, ctx->rd_tcnt, (size_t)std::max(nc, 1) * tiles * 4))) return s;
    if ((s = ensure(ctx, ctx->rd_cnum, (size_t)(d + 1) * 8))) return s;
    if (d > 16 && nc > 0 && (s = ensure(ctx, ctx->rd_xn, (size_t)N * d * 8))) return s;
    uint32_t* keys = (uint32_t*)ctx->rd_keys.p;
    uint64_t* k0 = (uint64_t*)ctx->rd_k0.p;
    uint64_t* k1 = (uint64_t*)ctx->rd_k1.p;
    uint32_t* hist = (uint32_t*)ctx->rd_hist.p;
    uint32_t* tcnt = (uint32_t*)ctx->rd_tcnt.p;
    unsigned long long* cnum = (unsigned long long*)ctx->rd_cnum.p;
    DevResult* dres = (DevResult*)ctx->res.p;
    auto grid_for = [](int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); };
    // full path: segmented 8-pass LSD radix sort of every corner's keys, then the tie-complete sweep
    auto full_sort = [&](cudaStream_t st) -> ddks_status {
        const int blocks = nc * tiles;
        uint64_t* src = nullptr;
        CU(cudaMemsetAsync(cnum, 0, (size_t)(d + 1) * 8, st));
        ddks_status rs = radix_sort_keys(ctx, k0, k1, N, nc, 0, hist, st, &src);
        if (rs) return rs;
        ddks::k_rd_count<<<blocks, ddks::RS_T, 0, st>>>(src, N, tiles, tcnt);
        ddks::k_rd_sweep<<<blocks, ddks::RS_T, 0, st>>>(src, N, tiles, n_P, n_Q, tcnt, cnum);
        CHECK_LAUNCH();
        ctx->launches += 2;
        return DDKS_OK;
    };
    // bucket-pruned sweep (default): workspace, and the known-zero state of the bucket counts -- k_rdb_cand /
    // k_rdb_finish re-zero every bucket they read, so after a completed call the first rdb_zero bytes of the buffer
    // are known zero (no memset of nb * 8 bytes); the memset this implies is part of the call graph and its key
    const bool pruned = !(ctx->flags & DDKS_FLAG_RDKS_FULL_SORT);
    int nbk = 256;
    while (nbk < N / rdb_bucket_div(N) && nbk < (1 << 20)) nbk <<= 1;
    const double scale = (double)nbk / (std::sqrt((double)d) * (1.0 + 1e-9));
    const size_t nb = (size_t)nc * nbk;
    const int nch = (nbk + ddks::RDB_CH - 1) / ddks::RDB_CH;
    const int cbytes = nbk / 8;  // the compaction's SMEM bitmap of one segment
    size_t zero = 0, rdb_clean_bytes = 0;
    if (nc > 0 && pruned) {
        if ((s = ensure(ctx, ctx->rdb_cnt, nb * 8))) return s;
        if ((s = ensure(ctx, ctx->rdb_pst, nb * 8))) return s;
        if ((s = ensure(ctx, ctx->rdb_coff, nb * 4))) return s;
        if ((s = ensure(ctx, ctx->rdb_fill, nb * 4))) return s;
        if ((s = ensure(ctx, ctx->rdb_bits, nb / 8))) return s;
        if ((s = ensure(ctx, ctx->rdb_clist, nb * 4))) return s;
        if ((s = ensure(ctx, ctx->rdb_csum, ((size_t)nc * nch + nc) * 8))) return s;
        zero = ctx->rdb_zero_p == ctx->rdb_cnt.p ? ctx->rdb_zero : 0;
        ctx->rdb_zero_p = nullptr;  // until this call completes
        rdb_clean_bytes = std::max(zero, nb * 8);
        if (cbytes > 48 * 1024)
            CU(cudaFuncSetAttribute(ddks::k_rdb_compact, cudaFuncAttributeMaxDynamicSharedMemorySize, cbytes));
    }
    if ((s = ensure_host(ctx, sizeof(DevResult) + (size_t)(d + 1) * 8))) return s;
    DevResult* hres = (DevResult*)ctx->host_pinned;
    uint64_t* hc = (uint64_t*)((char*)ctx->host_pinned + sizeof(DevResult));
    auto enq = [&](cudaStream_t st) -> ddks_status {
        ddks_status s;
        const void *dP, *dQ;
        if ((s = stage_input(ctx, P, (size_t)n_P * d * 4, ctx->raw_a, st, &dP))) return s;
        if ((s = stage_input(ctx, Q, (size_t)n_Q * d * 4, ctx->raw_b, st, &dQ))) return s;
        CU(cudaMemsetAsync(dres, 0, sizeof(DevResult), st));
        CU(cudaMemsetAsync(keys, 0xff, (size_t)d * 4, st));
        CU(cudaMemsetAsync(keys + d, 0, (size_t)d * 4, st));
        CU(cudaMemsetAsync(cnum, 0, (size_t)(d + 1) * 8, st));
        const int gy = std::min(d, 1024);
        const int gx = (int)std::max<int64_t>(1, std::min<int64_t>((N + 1023) / 1024, std::max(1, 296 / gy)));
        if (d <= 8 && ((((uintptr_t)dP | (uintptr_t)dQ) & 15) == 0)) {  // float4 rows-in-fours
            const int gv = (int)std::max<int64_t>(1, std::min<int64_t>((N / 4 + 255) / 256, ddks::MINMAX_BLOCKS));
            switch (d) {
#define MMV(D) case D: ddks::k_minmax_vec<D><<<gv, 256, 0, st>>>((const float*)dP, n_P, (const float*)dQ, n_Q, keys, D, 1, &dres->flag); break;
                MMV(1) MMV(2) MMV(3) MMV(4) MMV(5) MMV(6) MMV(7) MMV(8)
#undef MMV
            }
        } else {
            ddks::k_rd_minmax<<<dim3(gx, gy), 256, 0, st>>>(
                (const float*)dP, n_P, (const float*)dQ, n_Q, d, keys, &dres->flag);
        }
        CHECK_LAUNCH();
        ctx->launches++;
        // small d: NormalizeData is fused into the key kernel (x' recomputed per corner, no N x d f64 round trip);
        // large d (the paper's d = 1000 shape): normalise once, the key kernel reads x'
        const double* xn = nullptr;
        if (d > 16 && nc > 0) {
            ddks::k_rd_normalize<<<grid_for(N * d), 256, 0, st>>>((const float*)dP, n_P, (const float*)dQ, n_Q, d,
                                                                  keys, (double*)ctx->rd_xn.p);
            CHECK_LAUNCH();
            ctx->launches++;
            xn = (const double*)ctx->rd_xn.p;
        }
        if (nc > 0 && !pruned) {
            launch_rd_keys((const float*)dP, (const float*)dQ, xn, N, n_P, d, keys, (int)cb, (int)ce, k0, nullptr, 0,
                           0.0, st);
            CHECK_LAUNCH();
            ctx->launches++;
            if ((s = full_sort(st))) return s;
        } else if (nc > 0) {
            // bucket-pruned sweep: bucket counts, exact bucket-end values, sort only the buckets that can beat them
            uint32_t* bcnt = (uint32_t*)ctx->rdb_cnt.p;
            int32_t* clist = (int32_t*)ctx->rdb_clist.p;
            if (zero < nb * 8) CU(cudaMemsetAsync((uint8_t*)bcnt + zero, 0, nb * 8 - zero, st));
            // distance keys and their bucket counts in one pass (NormalizeData fused); profiled: the call's dominant
            // kernel, bound by L2 RED throughput (one bucket RED per key)
            std::pair<cudaEvent_t, cudaEvent_t> pev;
            if ((s = prof_begin(ctx, st, &pev))) return s;
            launch_rd_keys((const float*)dP, (const float*)dQ, xn, N, n_P, d, keys, (int)cb, (int)ce, k0, bcnt, nbk,
                           scale, st);
            if ((s = prof_end(ctx, st, pev, (uint64_t)nc * (uint64_t)N))) return s;
            uint64_t* csum = (uint64_t*)ctx->rdb_csum.p;
            uint32_t* segc = (uint32_t*)(csum + (size_t)nc * nch);
            CU(cudaMemsetAsync(segc, 0, (size_t)nc * 8, st));
            ddks::k_rdb_reduce<<<dim3(nch, nc), 256, 0, st>>>(bcnt, nbk, csum);
            ddks::k_rdb_chunk_scan<<<nc, 256, 0, st>>>(csum, nch);
            ddks::k_rdb_down<<<dim3(nch, nc), 256, 0, st>>>(bcnt, nbk, csum, n_P, n_Q, (uint2*)ctx->rdb_pst.p, cnum);
            ddks::k_rdb_cand<<<grid_for((int64_t)nb), 256, 0, st>>>(bcnt, (const uint2*)ctx->rdb_pst.p, nc, nbk, n_P,
                                                                    n_Q, cnum, (uint32_t*)ctx->rdb_coff.p,
                                                                    (uint32_t*)ctx->rdb_fill.p,
                                                                    (uint32_t*)ctx->rdb_bits.p, clist, segc);
            // compaction: ~2 CTAs per SM in all, split over the segments; the segment's bitmap in dynamic SMEM
            const int64_t cchunks = std::max<int64_t>(1, std::min<int64_t>((148 * DDKS_RDB_CPS + nc - 1) / nc,
                                                                           (N + ddks::RDB_CT - 1) / ddks::RDB_CT));
            ddks::k_rdb_compact<<<dim3((unsigned)cchunks, nc), ddks::RDB_CT, cbytes, st>>>(
                k0, N, nbk, scale, (const uint32_t*)ctx->rdb_bits.p, (const uint32_t*)ctx->rdb_coff.p,
                (uint32_t*)ctx->rdb_fill.p, k1);
            ddks::k_rdb_finish<<<dim3(std::max(1, std::min(1024, (148 * 4 + nc - 1) / nc)), nc), 256, 0, st>>>(
                k1, N, nbk, bcnt, (const uint2*)ctx->rdb_pst.p, (const uint32_t*)ctx->rdb_coff.p, clist, segc, n_P,
                n_Q, cnum, &dres->flag);
            CHECK_LAUNCH();
            ctx->launches += 7;
        }
        CU(cudaMemcpyAsync(hres, dres, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
        CU(cudaMemcpyAsync(hc, cnum, (size_t)std::max(nc, 0) * 8, cudaMemcpyDeviceToHost, st));
        return DDKS_OK;
    };
    const std::vector<uint64_t> key{(uint64_t)(uintptr_t)P, (uint64_t)(uintptr_t)Q, (uint64_t)n_P, (uint64_t)n_Q,
                                    (uint64_t)d, (uint64_t)ctx->flags, zero >= nb * 8 ? ~0ull : (uint64_t)zero};
    if ((s = run_call(ctx, ctx->cg_rdks, key, graph_input_ok(P) && graph_input_ok(Q), st, enq))) return s;
    CU(cudaStreamSynchronize(st));
    if ((s = collect_profile(ctx))) return s;
    if (nc > 0 && pruned && !(hres->flag & 256u)) {  // every bucket was read and re-zeroed
        ctx->rdb_zero_p = ctx->rdb_cnt.p;
        ctx->rdb_zero = rdb_clean_bytes;
    }
    if (nc > 0 && pruned && (hres->flag & 256u)) {  // a candidate bucket too large for SMEM: sort everything
        if ((s = full_sort(st))) return s;
        CU(cudaMemcpyAsync(hc, cnum, (size_t)nc * 8, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
    }
    if (ctx->comm) {
        NC(ncclAllReduce(&dres->flag, &dres->flag, 1, ncclUint32, ncclMax, ctx->comm, st));
        CU(cudaMemcpyAsync(&hres->flag, &dres->flag, 4, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
    }
    if (hres->flag & 1u) return fail(ctx, DDKS_ERR_NONFINITE, "non-finite coordinate in input");
    uint64_t best = 0;
    for (int c = 0; c < nc; ++c) best = std::max<uint64_t>(best, hc[c]);
    uint64_t arg = ~0ull;
    if (ctx->comm) {
        hres->num = best;
        CU(cudaMemcpyAsync(&dres->num, &hres->num, 8, cudaMemcpyHostToDevice, st));
        NC(ncclAllReduce(&dres->num, &dres->num, 1, ncclUint64, ncclMax, ctx->comm, st));
        CU(cudaMemcpyAsync(&hres->num, &dres->num, 8, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        best = hres->num;
    }
    for (int c = 0; c < nc; ++c)
        if (hc[c] == best) { arg = (uint64_t)(cb + c); break; }
    if (ctx->comm) {
        hres->arg = arg;
        CU(cudaMemcpyAsync(&dres->arg, &hres->arg, 8, cudaMemcpyHostToDevice, st));
        NC(ncclAllReduce(&dres->arg, &dres->arg, 1, ncclUint64, ncclMin, ctx->comm, st));
        CU(cudaMemcpyAsync(&hres->arg, &dres->arg, 8, cudaMemcpyDeviceToHost, st));
        CU(cudaStreamSynchronize(st));
        arg = hres->arg;
    }
    out->num = best;
    out->den = (uint64_t)n_P * (uint64_t)n_Q;
    out->D = (double)best / (double)out->den;
    out->argmax_origin = (int64_t)arg;
    return DDKS_OK;
}

}  // extern "C"
