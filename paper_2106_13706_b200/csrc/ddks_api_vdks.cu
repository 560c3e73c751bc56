// ddks_api_vdks.cu — C-ABI entry ddks_vdks (include/ddks.h; §2.2.2, Alg. 1).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>

#include "ddks_internal.h"
#include "ddks_vdks.cuh"

using namespace ddks_host;

extern "C" {

// ------------------------------------------------------------------------------------- vdKS (Alg. 1)
// Points sharded across ranks for the voxel histogram (NCCL all-reduce(sum) of the grid counts), voxels sharded
// for the orthant sums (all-reduce(max)); min/max keys all-reduced (min / max) before voxelisation.
ddks_status ddks_vdks(ddks_ctx* ctx, const float* P, int64_t n_P, const float* Q, int64_t n_Q, int32_t d, int64_t k,
                      void* stream, ddks_result* out) {
    if (!ctx) return DDKS_ERR_INVALID_ARGUMENT;
    ctx->err.clear();
    if (!out) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "null out");
    ddks_status s = check_sizes(ctx, n_P, n_Q, d);
    if (s) return s;
    if (!P || !Q) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "null argument");
    if (k < 1) return fail(ctx, DDKS_ERR_INVALID_ARGUMENT, "k=%lld < 1", (long long)k);
    int64_t V = 1;
    for (int m = 0; m < d; ++m) {
        if (V > (int64_t(1) << 30) / k) return fail(ctx, DDKS_ERR_TOO_LARGE, "k^d > 2^30 voxels");
        V *= k;
    }
    if ((s = bind_device(ctx))) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t N = n_P + n_Q;
    // slab scans: L = k^J voxels per slab, the largest J with L <= VS_MAX_L (J = 0: k > 4096, line passes only)
    int J = 0;
    int64_t L = 1;
    if (k == 1) {
        J = d;
    } else {
        for (int j = 1; j <= d && L * k <= ddks::VS_MAX_L; ++j) J = j, L *= k;
    }
    const int64_t NS = V / L;
    const bool use_list = ctx->world <= 1;  // one rank: orthants over the compact filled-voxel list
    const int64_t n_list_max = std::min<int64_t>(V, N);
    if ((s = ensure(ctx, ctx->vox_keys, 16 * 4))) return s;
    if ((s = ensure(ctx, ctx->vox_cnt, (size_t)V * 8))) return s;
    if ((s = ensure(ctx, ctx->vox_S, (size_t)V * 8))) return s;
    if ((s = ensure(ctx, ctx->vox_fill, (size_t)V))) return s;
    if ((s = ensure(ctx, ctx->vox_slab, (size_t)(n_list_max + 1) * 4))) return s;
    uint32_t* keys = (uint32_t*)ctx->vox_keys.p;
    uint32_t* cnt = (uint32_t*)ctx->vox_cnt.p;
    int64_t* S = (int64_t*)ctx->vox_S.p;
    uint8_t* fill = (uint8_t*)ctx->vox_fill.p;
    uint32_t* n_list = (uint32_t*)ctx->vox_slab.p;
    uint32_t* list = use_list ? n_list + 1 : nullptr;
    DevResult* dres = (DevResult*)ctx->res.p;
    DevResult* hres = (DevResult*)ctx->host_pinned;
    // the counts: the call needs [0, 8 V) zero; earlier calls' slab scans left a known-zero prefix of the buffer (the
    // memset this implies is part of the call graph, so the known-zero state is part of its key)
    const size_t zero = ctx->vox_zero_p == ctx->vox_cnt.p ? ctx->vox_zero : 0;
    ctx->vox_zero_p = nullptr;  // until this call completes
    auto enq = [&](cudaStream_t st) -> ddks_status {
        ddks_status s;
        const void *dP, *dQ;
        if ((s = stage_input(ctx, P, (size_t)n_P * d * 4, ctx->raw_a, st, &dP))) return s;
        if ((s = stage_input(ctx, Q, (size_t)n_Q * d * 4, ctx->raw_b, st, &dQ))) return s;
        ddks::k_vox_init<<<1, 32, 0, st>>>(keys, (unsigned long long*)dres, use_list ? n_list : nullptr);
        CHECK_LAUNCH();
        ctx->launches++;
        if (zero < (size_t)V * 8) CU(cudaMemsetAsync((uint8_t*)cnt + zero, 0, (size_t)V * 8 - zero, st));
        // the points are read in place (no pack): k_minmax validates them and k_vox_hist voxelises them
        int64_t pb, pe;
        ddks_shard_range(N, ctx->world, ctx->rank, &pb, &pe);
        const int blk = 256;
        auto grid_for = [](int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); };
        const bool aligned = (((uintptr_t)dP | (uintptr_t)dQ) & 15) == 0;
        const bool whole = pb == 0 && pe == N && aligned;  // one rank holds all points: vectorised kernels
        if (whole) {
            const int gv = (int)std::max<int64_t>(1, std::min<int64_t>((N / 4 + 255) / 256, ddks::MINMAX_BLOCKS));
            const int val = !(ctx->flags & DDKS_FLAG_NO_VALIDATE);
            switch (d) {
    #define MMV(D) case D: ddks::k_minmax_vec<D><<<gv, blk, 0, st>>>((const float*)dP, n_P, (const float*)dQ, n_Q, keys, 8, val, &dres->flag); break;
                MMV(1) MMV(2) MMV(3) MMV(4) MMV(5) MMV(6) MMV(7) MMV(8)
    #undef MMV
            }
            CHECK_LAUNCH();
            ctx->launches++;
        } else if (pe > pb) {
            ddks::k_minmax<<<(int)std::max<int64_t>(1, std::min<int64_t>((pe - pb + 255) / 256, 148 * 8)), blk, 0, st>>>(
                (const float*)dP, (const float*)dQ, n_P, pb, pe, d, keys, !(ctx->flags & DDKS_FLAG_NO_VALIDATE),
                &dres->flag);
            CHECK_LAUNCH();
            ctx->launches++;
        }
        if (ctx->comm) {
            NC(ncclAllReduce(keys, keys, 8, ncclUint32, ncclMin, ctx->comm, st));
            NC(ncclAllReduce(keys + 8, keys + 8, 8, ncclUint32, ncclMax, ctx->comm, st));
        }
        // profiled: the voxel histogram (the call's dominant kernel, bound by L2 RED throughput), one RED per point
        std::pair<cudaEvent_t, cudaEvent_t> pev;
        if ((s = prof_begin(ctx, st, &pev))) return s;
        if (whole) {
            const int gh = (int)std::max<int64_t>(1, std::min<int64_t>((N / 4 + 255) / 256, 148 * 8));
            switch (d) {
    #define VH(D) case D: ddks::k_vox_hist_vec<D><<<gh, blk, 0, st>>>((const float*)dP, n_P, (const float*)dQ, n_Q, keys, (int)k, cnt); break;
                VH(1) VH(2) VH(3) VH(4) VH(5) VH(6) VH(7) VH(8)
    #undef VH
            }
            CHECK_LAUNCH();
            ctx->launches++;
        } else if (pe > pb) {
            ddks::k_vox_hist<<<grid_for(pe - pb), blk, 0, st>>>((const float*)dP, (const float*)dQ, pb, pe, n_P, d, keys,
                                                                k, cnt);
            CHECK_LAUNCH();
            ctx->launches++;
        }
        if ((s = prof_end(ctx, st, pev, (uint64_t)(whole ? N : std::max<int64_t>(pe - pb, 0))))) return s;
        if (ctx->comm) {
            NC(ncclAllReduce(cnt, cnt, (size_t)V * 2, ncclUint32, ncclSum, ctx->comm, st));
            NC(ncclAllReduce(&dres->flag, &dres->flag, 1, ncclUint32, ncclMax, ctx->comm, st));
        }
        const int lg = (k & (k - 1)) == 0 ? __builtin_ctzll((unsigned long long)k) : -1;
        int64_t stride = 1;  // first dimension not yet scanned: stride k^m
        int m0 = 0;
        if (J > 0) {
            const size_t smb = (size_t)L * 9;
            if (smb > 48 * 1024)
                CU(cudaFuncSetAttribute(ddks::k_vox_prefix_slab, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smb));
            ddks::k_vox_prefix_slab<<<(unsigned)NS, ddks::VS_SLAB_T, smb, st>>>(cnt, 1, (int)k, lg, J, (int)L, n_P, n_Q,
                                                                                S, fill, list, n_list);
            CHECK_LAUNCH();
            ctx->launches++;
            m0 = J, stride = L;
            if (J < d && NS <= ddks::VS_OUTER_MAX_NS) {
                const size_t smo = (size_t)NS * ddks::VS_OUTER_CW * 8;
                if (smo > 48 * 1024)
                    CU(cudaFuncSetAttribute(ddks::k_vox_outer, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smo));
                ddks::k_vox_outer<<<(unsigned)((L + ddks::VS_OUTER_CW - 1) / ddks::VS_OUTER_CW), 256, smo, st>>>(
                    S, (int)k, (int)L, (int)NS, d - J);
                CHECK_LAUNCH();
                ctx->launches++;
                m0 = d;
            }
        }
        for (int m = m0; m < d; ++m, stride *= k) {
            ddks::k_prefix_line<<<grid_for(V / k), blk, 0, st>>>(S, V, k, stride, m == 0 ? cnt : nullptr, n_P, n_Q, fill);
            CHECK_LAUNCH();
            ctx->launches++;
        }
        if (J == 0 && use_list) {  // the line passes build no list: orthants over the fill bytes
            list = nullptr;
        }
        int64_t vb, ve;
        ddks_shard_range(V, ctx->world, ctx->rank, &vb, &ve);
        if (ve > vb) {
            unsigned long long* num = &dres->num;
            const int g = grid_for(list ? n_list_max : ve - vb);
            switch (d) {
    #define VO(D) case D: ddks::k_vox_orthants<D><<<g, blk, 0, st>>>(fill, list, n_list, S, vb, ve, (int)k, lg, num); break;
                VO(1) VO(2) VO(3) VO(4) VO(5) VO(6) VO(7) VO(8)
    #undef VO
            }
            CHECK_LAUNCH();
            ctx->launches++;
        }
        if (ctx->comm) NC(ncclAllReduce(&dres->num, &dres->num, 1, ncclUint64, ncclMax, ctx->comm, st));
        CU(cudaMemcpyAsync(hres, dres, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
        return DDKS_OK;
    };
    const std::vector<uint64_t> key{(uint64_t)(uintptr_t)P, (uint64_t)(uintptr_t)Q, (uint64_t)n_P, (uint64_t)n_Q,
                                    (uint64_t)d, (uint64_t)k, (uint64_t)ctx->flags,
                                    zero >= (size_t)V * 8 ? ~0ull : (uint64_t)zero};
    if ((s = run_call(ctx, ctx->cg_vdks, key, graph_input_ok(P) && graph_input_ok(Q), st, enq))) return s;
    CU(cudaStreamSynchronize(st));
    if ((s = collect_profile(ctx))) return s;
    if (J > 0) {  // every slab zeroed its counts: [0, max(zero, 8 V)) is zero again
        ctx->vox_zero_p = ctx->vox_cnt.p;
        ctx->vox_zero = std::max(zero, (size_t)V * 8);
    }
    if (hres->flag & 1u) return fail(ctx, DDKS_ERR_NONFINITE, "non-finite coordinate in input");
    out->num = hres->num;
    out->den = (uint64_t)n_P * (uint64_t)n_Q;
    out->D = (double)out->num / (double)out->den;
    out->argmax_origin = -1;
    return DDKS_OK;
}

}  // extern "C"
