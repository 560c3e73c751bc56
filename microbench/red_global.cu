// Global RED.ADD.u32 throughput into an L2-resident count array, the access pattern of the vdKS voxel histogram
// (k_vox_hist_vec) separated from its loads and voxel arithmetic: ids are precomputed on the host.
//   (a) uniform random voxel ids over k^d = 16^5 voxels x 2 labels (8 MB of counts);
//   (b) the C5 voxel ids: 2 x 10^6 5-d points, P ~ N(0, I), Q ~ 0.9 N(0, I) + 0.1 N(0.5, 0.25 I), normalised by the
//       pooled min / max and cut into 16 cells per dimension (the hot central voxels collide);
//   (c) as (b) with the ids sorted (every warp's REDs hit few addresses: the same-address serialisation bound).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_global red_global.cu && ./red_global
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>
#include <cuda_runtime.h>

__global__ void k_red(const uint32_t* __restrict__ ids, int n, uint32_t* __restrict__ cnt) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) atomicAdd(&cnt[ids[i]], 1u);
}
// four ids per thread per iteration (one 16-byte load): more REDs in flight per thread
__global__ void k_red4(const uint4* __restrict__ ids, int n4, uint32_t* __restrict__ cnt) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += gridDim.x * blockDim.x) {
        const uint4 v = ids[i];
        atomicAdd(&cnt[v.x], 1u);
        atomicAdd(&cnt[v.y], 1u);
        atomicAdd(&cnt[v.z], 1u);
        atomicAdd(&cnt[v.w], 1u);
    }
}

static float time_red(const uint32_t* d_ids, int n, uint32_t* d_cnt, size_t cnt_words, int variant = 0, int blocks = 148 * 8) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 20; ++rep) {
        cudaMemset(d_cnt, 0, cnt_words * 4);
        cudaEventRecord(e0);
        if (variant == 0) k_red<<<blocks, 256>>>(d_ids, n, d_cnt);
        else k_red4<<<blocks, 256>>>(reinterpret_cast<const uint4*>(d_ids), n / 4, d_cnt);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
    }
    return best * 1e3f;
}

int main() {
    const int n = 2000000, d = 5, k = 16;
    const size_t V = 1u << 20, words = 2 * V;
    std::mt19937_64 rng(4);
    std::normal_distribution<double> nd(0.0, 1.0);
    std::uniform_real_distribution<double> ud(0.0, 1.0);
    std::vector<float> x((size_t)n * d);
    for (int i = 0; i < n; ++i) {
        const bool q = i >= n / 2, mix = q && ud(rng) < 0.1;
        for (int m = 0; m < d; ++m) x[(size_t)i * d + m] = (float)(mix ? 0.5 + 0.5 * nd(rng) : (q ? 0.9 : 1.0) * nd(rng));
    }
    double mn[d], mx[d];
    for (int m = 0; m < d; ++m) mn[m] = 1e300, mx[m] = -1e300;
    for (int i = 0; i < n; ++i)
        for (int m = 0; m < d; ++m) mn[m] = std::min(mn[m], (double)x[(size_t)i * d + m]), mx[m] = std::max(mx[m], (double)x[(size_t)i * d + m]);
    std::vector<uint32_t> ids_c5(n), ids_uni(n);
    std::uniform_int_distribution<uint32_t> vd(0, (uint32_t)V - 1);
    for (int i = 0; i < n; ++i) {
        uint32_t flat = 0, stride = 1;
        for (int m = 0; m < d; ++m) {
            int c = (int)std::floor((x[(size_t)i * d + m] - mn[m]) / (mx[m] - mn[m]) * k);
            c = std::min(std::max(c, 0), k - 1);
            flat += (uint32_t)c * stride;
            stride *= k;
        }
        const uint32_t q = i >= n / 2;
        ids_c5[i] = 2 * flat + q;
        ids_uni[i] = 2 * vd(rng) + q;
    }
    std::vector<uint32_t> hot(V * 2, 0);
    for (uint32_t v : ids_c5) hot[v]++;
    const uint32_t hottest = *std::max_element(hot.begin(), hot.end());
    size_t distinct = 0;
    for (uint32_t c : hot) distinct += c != 0;
    std::vector<uint32_t> ids_sorted = ids_c5;
    std::sort(ids_sorted.begin(), ids_sorted.end());
    uint32_t *d_ids, *d_cnt;
    cudaMalloc(&d_ids, (size_t)n * 4);
    cudaMalloc(&d_cnt, words * 4);
    const char* names[3] = {"uniform random ids", "C5 voxel ids (pooled order)", "C5 voxel ids sorted"};
    const std::vector<uint32_t>* sets[3] = {&ids_uni, &ids_c5, &ids_sorted};
    printf("n = %d REDs into %zu u32 counts (%.1f MB); C5: %zu distinct (voxel, label) cells, hottest %u\n", n, words,
           words * 4 / 1e6, distinct, hottest);
    for (int s = 0; s < 3; ++s) {
        cudaMemcpy(d_ids, sets[s]->data(), (size_t)n * 4, cudaMemcpyHostToDevice);
        for (int variant = 0; variant < 2; ++variant)
            for (int blocks : {148 * 4, 148 * 8, 148 * 16}) {
                const float us = time_red(d_ids, n, d_cnt, words, variant, blocks);
                printf("%-30s %s grid %5d  %8.2f us  %.3e RED/s\n", names[s], variant ? "4/thread" : "1/thread", blocks,
                       us, n / (us * 1e-6));
            }
    }
    // steady-state peak: 12e6 uniform REDs (the rdKS key pass's count) into count arrays of several sizes
    {
        const int n2 = 12000000;
        uint32_t* d_ids2;
        cudaMalloc(&d_ids2, (size_t)n2 * 4);
        for (size_t w2 : {(size_t)1 << 21, (size_t)6291456, (size_t)1 << 24}) {
            std::vector<uint32_t> ids2(n2);
            std::uniform_int_distribution<uint32_t> wd(0, (uint32_t)w2 - 1);
            for (auto& v : ids2) v = wd(rng);
            uint32_t* d_cnt2;
            cudaMalloc(&d_cnt2, w2 * 4);
            cudaMemcpy(d_ids2, ids2.data(), (size_t)n2 * 4, cudaMemcpyHostToDevice);
            for (int variant = 0; variant < 2; ++variant) {
                const float us = time_red(d_ids2, n2, d_cnt2, w2, variant, 148 * 16);
                printf("12e6 uniform REDs into %6.1f MB  %s  %8.2f us  %.3e RED/s\n", w2 * 4 / 1e6,
                       variant ? "4/thread" : "1/thread", us, n2 / (us * 1e-6));
            }
            cudaFree(d_cnt2);
        }
    }
    return 0;
}
