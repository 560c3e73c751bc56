// ddks_common.cuh — device helpers shared by every kernel header of libddks.so (all inline: safe to include from
// several translation units): order-preserving float keys, the TMA-bulk / mbarrier / SMEM-atomic PTX wrappers,
// warp and block scans, and the radix-sort tile geometry.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

// Device-side bounds checks, compiled in with -DDDKS_DEBUG (build.py: DDKS_DEBUG=1). compute-sanitizer is not
// available on the GPU pool, so the debug build's asserts (run under the whole GPU test suite) stand in for memcheck.
#ifdef DDKS_DEBUG
#include <cassert>
#define DDKS_ASSERT(c) assert(c)
#else
#define DDKS_ASSERT(c) ((void)0)
#endif

namespace ddks {

template <int D> __host__ __device__ constexpr int padded_dim() { return D <= 4 ? 4 : 8; }

// order-preserving uint32 key of a float (after -0 -> +0 canonicalisation) and its inverse
__device__ __forceinline__ uint32_t f32_key(float f) {
    const uint32_t b = __float_as_uint(f);
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __forceinline__ float key_f32(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

// ----------------------------------------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// DDKS_MBAR_HINT_NS > 0 builds the wait with a suspend-time hint (a waiting warp sleeps until the phase completes or
// the hint expires instead of re-issuing try_wait every ~70 cycles; at C5 those re-issues were 13 % of the kd count's
// executed instructions). Measured: neutral at C5 / C3 / C2 (microbench/r2_hint_sweep.sh) but C4 +8 % (1.427 ->
// 1.547 ms: 4096 short CTAs that each wait for their first tiles; microbench/r2_c4hint.sh), so the default is off.
#ifndef DDKS_MBAR_HINT_NS
#define DDKS_MBAR_HINT_NS 0
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#if DDKS_MBAR_HINT_NS == 0
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "DDKS_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra DDKS_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
    return;
#endif
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "DDKS_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra DDKS_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity), "n"(DDKS_MBAR_HINT_NS)
        : "memory");
}
// 1-D bulk copy global -> shared through the TMA engine, completion counted on an mbarrier (bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// FP32 ordered compare -> 1.0f / 0.0f (SASS FSET.BF). No .ftz: denormals compare exactly (R6).
template <bool GT> __device__ __forceinline__ float cmp_bit(float x, float o) {
    float r;
    if constexpr (GT) asm("set.gt.f32.f32 %0, %1, %2;" : "=f"(r) : "f"(x), "f"(o));
    else              asm("set.ge.f32.f32 %0, %1, %2;" : "=f"(r) : "f"(x), "f"(o));
    return r;
}
// No "memory" clobber: the counters are only read after a __syncthreads() (a compiler and hardware fence), and the
// point tiles the hot loop loads are disjoint from them, so ptxas may hoist the next point's LDS above these REDs.
__device__ __forceinline__ void red_add_shared(uint32_t addr, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v));
}

__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const uint64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

// ------------------------------------------------------------------------------------ segmented LSD radix sort
constexpr int RS_T = 256, RS_ITEMS = 16, RS_TILE = RS_T * RS_ITEMS, RS_WARPS = RS_T / 32;

// Exclusive scan over a 256-thread block (one value per thread; warp shuffles + one warp over the 8 warp totals).
// *total (if given) receives the block sum. Contains __syncthreads().
__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t v, uint32_t* total = nullptr) {
    __shared__ uint32_t wsum[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        uint32_t s = lane < 8 ? wsum[lane] : 0u;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < 8) wsum[lane] = s;  // inclusive warp-total prefix
    }
    __syncthreads();
    if (total) *total = wsum[7];
    return x - v + (w ? wsum[w - 1] : 0u);
}

// 64-bit variant (packed (cP, cQ) pairs in the rdKS bucket scans)
__device__ __forceinline__ uint64_t block_excl_scan256_u64(uint64_t v, uint64_t* total = nullptr) {
    __shared__ uint64_t wsum64[8];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint64_t x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    __syncthreads();
    if (lane == 31) wsum64[w] = x;
    __syncthreads();
    if (w == 0) {
        uint64_t t = lane < 8 ? wsum64[lane] : 0ull;
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < 8) wsum64[lane] = t;
    }
    __syncthreads();
    if (total) *total = wsum64[7];
    return x - v + (w ? wsum64[w - 1] : 0ull);
}

}  // namespace ddks
