// RED.shared throughput when a thread's consecutive increments hit the same word vs different words.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_same_addr red_same_addr.cu && ./red_same_addr
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void red_add(uint32_t addr, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v));
}

// mode 0: every op a different word (round robin over NW words per thread); mode k: the same word k times in a row
template <int NW>
__global__ void k(int iters, int repeat, unsigned long long* cyc, uint32_t* sink) {
    __shared__ uint32_t cnt[NW * 256];
    for (int i = threadIdx.x; i < NW * 256; i += blockDim.x) cnt[i] = 0;
    __syncthreads();
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(cnt) + 4u * threadIdx.x;
    unsigned long long t0 = clock64();
    int w = 0, r = 0;
#pragma unroll 16
    for (int i = 0; i < iters; ++i) {
        red_add(base + 4u * 256u * (uint32_t)w, 1u);
        if (++r == repeat) { r = 0; w = (w + 1) % NW; }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) atomicAdd(cyc, t1 - t0);
    if (cnt[threadIdx.x] == 12345) sink[0] = 1;
}

int main() {
    unsigned long long* cyc;
    uint32_t* sink;
    cudaMalloc(&cyc, 8);
    cudaMalloc(&sink, 4);
    const int iters = 1 << 16, blocks = 148 * 2, threads = 256;
    for (int rep : {1, 2, 4, 8, 64}) {
        cudaMemset(cyc, 0, 8);
        k<8><<<blocks, threads>>>(iters, rep, cyc, sink);
        cudaDeviceSynchronize();
        unsigned long long c;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        const double cyc_per_block = (double)c / blocks;
        // lanes per clock per SM (2 blocks per SM resident)
        const double lanes = (double)iters * threads * 2 / cyc_per_block;
        printf("same word %2d times in a row: %.2f RED lanes/clk/SM (%.1f cycles per block)\n", rep, lanes, cyc_per_block);
    }
    return 0;
}
