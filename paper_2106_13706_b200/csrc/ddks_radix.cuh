// ddks_radix.cuh — segmented, stable LSD radix sort of 64-bit keys, 8-bit digits (SURVEY §8f NEXT-4 sort, and the
// x0 ordering of the exact statistic). Included by ONE translation unit (ddks_api.cu); others call
// ddks_host::radix_sort_keys (ddks_internal.h).
//   k_rs_hist    per 4096-key tile digit histogram;
//   k_rs_scan    per segment: tile-major running offsets + digit-base scan (4 threads per digit);
//   k_rs_scatter stable scatter: warp __match_any_sync ranks + per-warp digit counters, regrouped by digit in SMEM,
//                then written with consecutive threads on consecutive addresses (coalesced).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "ddks_common.cuh"

namespace ddks {

// hist[(seg * tiles + tile) * 256 + digit]
__global__ void __launch_bounds__(RS_T) k_rs_hist(const uint64_t* __restrict__ in, int64_t N, int tiles, int shift,
                                                  uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[256];
    const int seg = blockIdx.x / tiles, tile = blockIdx.x - seg * tiles;
    const int64_t base = (int64_t)seg * N + (int64_t)tile * RS_TILE;
    const int n = (int)min((int64_t)RS_TILE, N - (int64_t)tile * RS_TILE);
    h[threadIdx.x] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += RS_T) atomicAdd(&h[(uint32_t)(in[base + i] >> shift) & 255u], 1u);
    __syncthreads();
    hist[(int64_t)blockIdx.x * 256 + threadIdx.x] = h[threadIdx.x];
}

// In place: hist -> offsets within the segment, offs[tile][dig] = sum_{d' < dig} total[d'] + sum_{t' < tile} h[t'][dig].
// One CTA of 1024 threads per segment: thread (part, dig) owns a quarter of the tiles of one digit; tiles are read
// 16 at a time so the loads overlap.
constexpr int RS_SCAN_PARTS = 4;
__global__ void __launch_bounds__(256 * RS_SCAN_PARTS) k_rs_scan(uint32_t* __restrict__ hist, int tiles) {
    __shared__ uint32_t pt[RS_SCAN_PARTS][256];
    __shared__ uint32_t dbase[256];
    __shared__ uint32_t wtot[8];
    const int seg = blockIdx.x, dig = threadIdx.x & 255, part = threadIdx.x >> 8;
    const int lane = threadIdx.x & 31, w = (threadIdx.x >> 5) & 7;
    uint32_t* h = hist + (int64_t)seg * tiles * 256;
    const int per = (tiles + RS_SCAN_PARTS - 1) / RS_SCAN_PARTS;
    const int t_begin = min(tiles, part * per), t_end = min(tiles, t_begin + per);
    uint32_t run = 0;
    for (int t0 = t_begin; t0 < t_end; t0 += 16) {
        uint32_t v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = t0 + j < t_end ? h[(t0 + j) * 256 + dig] : 0u;
#pragma unroll
        for (int j = 0; j < 16; ++j) run += v[j];
    }
    pt[part][dig] = run;
    __syncthreads();
    uint32_t tot = 0, x = 0;
    if (part == 0) {
#pragma unroll
        for (int p = 0; p < RS_SCAN_PARTS; ++p) tot += pt[p][dig];
        x = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wtot[w] = x;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t r = 0;
        for (int i = 0; i < 8; ++i) {
            const uint32_t v = wtot[i];
            wtot[i] = r;
            r += v;
        }
    }
    __syncthreads();
    if (part == 0) dbase[dig] = x - tot + wtot[w];
    __syncthreads();
    run = dbase[dig];
    for (int p = 0; p < part; ++p) run += pt[p][dig];
    for (int t0 = t_begin; t0 < t_end; t0 += 16) {
        uint32_t v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = t0 + j < t_end ? h[(t0 + j) * 256 + dig] : 0u;
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (t0 + j < t_end) {
                h[(t0 + j) * 256 + dig] = run;
                run += v[j];
            }
    }
}

// Stable scatter of one tile: warp w ranks its 512 keys (rounds of 32, in tile order) with __match_any_sync and a
// per-warp digit counter; warps are then ordered by an exclusive scan of their counters per digit. The tile is
// first regrouped by digit in SMEM (local position = tile digit base + warp offset + rank) and then written out
// with consecutive threads on consecutive addresses of each digit's run (coalesced).
__global__ void __launch_bounds__(RS_T) k_rs_scatter(const uint64_t* __restrict__ in, uint64_t* __restrict__ out,
                                                     int64_t N, int tiles, int shift,
                                                     const uint32_t* __restrict__ offs) {
    __shared__ uint32_t wc[RS_WARPS][256];
    __shared__ uint32_t dbase[256];   // exclusive scan of the tile's digit counts
    __shared__ uint64_t stage[RS_TILE];
    const int seg = blockIdx.x / tiles, tile = blockIdx.x - seg * tiles;
    const int64_t sbase = (int64_t)seg * N;
    const int64_t base = sbase + (int64_t)tile * RS_TILE;
    const int n = (int)min((int64_t)RS_TILE, N - (int64_t)tile * RS_TILE);
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < RS_WARPS * 256; i += RS_T) (&wc[0][0])[i] = 0;
    __syncthreads();
    const uint32_t lt = (1u << lane) - 1u;
    uint64_t k[RS_ITEMS];
    uint32_t rank[RS_ITEMS], dg[RS_ITEMS];
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j) {
        const int idx = w * (RS_ITEMS * 32) + j * 32 + lane;
        const bool valid = idx < n;
        k[j] = valid ? in[base + idx] : 0ull;
        const uint32_t dig = valid ? ((uint32_t)(k[j] >> shift) & 255u) : 256u;
        dg[j] = dig;
        const uint32_t peers = __match_any_sync(0xffffffffu, dig);
        uint32_t b = 0;
        if (valid) b = wc[w][dig];
        __syncwarp();
        rank[j] = b + __popc(peers & lt);
        if (valid && (peers & lt) == 0) wc[w][dig] = b + __popc(peers);  // the group's lowest lane
        __syncwarp();
    }
    __syncthreads();
    {
        uint32_t run = 0;
#pragma unroll
        for (int ww = 0; ww < RS_WARPS; ++ww) {
            const uint32_t v = wc[ww][threadIdx.x];
            wc[ww][threadIdx.x] = run;
            run += v;
        }
        dbase[threadIdx.x] = block_excl_scan256(run);  // exclusive scan of the tile's digit counts
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < RS_ITEMS; ++j)
        if (dg[j] < 256u) stage[dbase[dg[j]] + wc[w][dg[j]] + rank[j]] = k[j];
    __syncthreads();
    const uint32_t* o = offs + (int64_t)blockIdx.x * 256;
    for (int i = threadIdx.x; i < n; i += RS_T) {
        const uint64_t key = stage[i];
        const uint32_t dig = (uint32_t)(key >> shift) & 255u;
        DDKS_ASSERT((int64_t)o[dig] + i - dbase[dig] < N);
        out[sbase + o[dig] + (uint32_t)i - dbase[dig]] = key;
    }
}

}  // namespace ddks
