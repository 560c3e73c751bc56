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
    const void *dP, *dQ;
    if ((s = stage_input(ctx, P, (size_t)n_P * d * 4, ctx->raw_a, st, &dP))) return s;
    if ((s = stage_input(ctx, Q, (size_t)n_Q * d * 4, ctx->raw_b, st, &dQ))) return s;
    if ((s = ensure(ctx, ctx->vox_keys, 16 * 4))) return s;
    if ((s = ensure(ctx, ctx->vox_cnt, (size_t)V * 8))) return s;
    if ((s = ensure(ctx, ctx->vox_S, (size_t)V * 8))) return s;
    uint32_t* keys = (uint32_t*)ctx->vox_keys.p;
    uint32_t* cnt = (uint32_t*)ctx->vox_cnt.p;
    int64_t* S = (int64_t*)ctx->vox_S.p;
    DevResult* dres = (DevResult*)ctx->res.p;
    DevResult* hres = (DevResult*)ctx->host_pinned;
    *hres = DevResult{0ull, ~0ull, 0ull, 0u, 0u};
    CU(cudaMemcpyAsync(dres, hres, sizeof(DevResult), cudaMemcpyHostToDevice, st));
    CU(cudaMemsetAsync(keys, 0xff, 8 * 4, st));
    CU(cudaMemsetAsync(keys + 8, 0, 8 * 4, st));
    CU(cudaMemsetAsync(cnt, 0, (size_t)V * 8, st));
    // the points are read in place (no pack): k_minmax validates them and k_vox_hist voxelises them
    int64_t pb, pe;
    ddks_shard_range(N, ctx->world, ctx->rank, &pb, &pe);
    const int blk = 256;
    auto grid_for = [](int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); };
    const bool aligned = (((uintptr_t)dP | (uintptr_t)dQ) & 15) == 0;
    if (pb == 0 && pe == N && aligned) {  // one rank holds all points: vectorised min / max
        const int gv = (int)std::max<int64_t>(1, std::min<int64_t>((N / 4 + 255) / 256, 148 * 8));
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
    if (pe > pb) {
        ddks::k_vox_hist<<<grid_for(pe - pb), blk, 0, st>>>((const float*)dP, (const float*)dQ, pb, pe, n_P, d, keys,
                                                            k, cnt);
        CHECK_LAUNCH();
        ctx->launches++;
    }
    if (ctx->comm) {
        NC(ncclAllReduce(cnt, cnt, (size_t)V * 2, ncclUint32, ncclSum, ctx->comm, st));
        NC(ncclAllReduce(&dres->flag, &dres->flag, 1, ncclUint32, ncclMax, ctx->comm, st));
    }
    int64_t stride = 1;
    for (int m = 0; m < d; ++m, stride *= k) {
        if (m == 0 && k <= 32 && (k & (k - 1)) == 0) {  // coalesced segmented warp scan of the k-voxel lines
            ddks::k_prefix_first<<<grid_for(V), blk, 0, st>>>(S, V, (int)k, cnt, n_P, n_Q);
        } else {
            ddks::k_prefix_line<<<grid_for(V / k), blk, 0, st>>>(S, V, k, stride, m == 0 ? cnt : nullptr, n_P, n_Q);
        }
        CHECK_LAUNCH();
        ctx->launches++;
    }
    int64_t vb, ve;
    ddks_shard_range(V, ctx->world, ctx->rank, &vb, &ve);
    if (ve > vb) {
        unsigned long long* num = &dres->num;
        const int g = grid_for(ve - vb);
        switch (d) {
            case 1: ddks::k_vox_orthants<1><<<g, blk, 0, st>>>(cnt, S, vb, ve, k, num); break;
            case 2: ddks::k_vox_orthants<2><<<g, blk, 0, st>>>(cnt, S, vb, ve, k, num); break;
            case 3: ddks::k_vox_orthants<3><<<g, blk, 0, st>>>(cnt, S, vb, ve, k, num); break;
            case 4: ddks::k_vox_orthants<4><<<g, blk, 0, st>>>(cnt, S, vb, ve, k, num); break;
            case 5: ddks::k_vox_orthants<5><<<g, blk, 0, st>>>(cnt, S, vb, ve, k, num); break;
            case 6: ddks::k_vox_orthants<6><<<g, blk, 0, st>>>(cnt, S, vb, ve, k, num); break;
            case 7: ddks::k_vox_orthants<7><<<g, blk, 0, st>>>(cnt, S, vb, ve, k, num); break;
            case 8: ddks::k_vox_orthants<8><<<g, blk, 0, st>>>(cnt, S, vb, ve, k, num); break;
        }
        CHECK_LAUNCH();
        ctx->launches++;
    }
    if (ctx->comm) NC(ncclAllReduce(&dres->num, &dres->num, 1, ncclUint64, ncclMax, ctx->comm, st));
    CU(cudaMemcpyAsync(hres, dres, sizeof(DevResult), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    if (hres->flag & 1u) return fail(ctx, DDKS_ERR_NONFINITE, "non-finite coordinate in input");
    out->num = hres->num;
    out->den = (uint64_t)n_P * (uint64_t)n_Q;
    out->D = (double)out->num / (double)out->den;
    out->argmax_origin = -1;
    return DDKS_OK;
}

}  // extern "C"
