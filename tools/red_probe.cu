// red_probe.cu — cost model of fire-and-forget L2 reductions (RED.ADD.U32)
// on the box's GPU: throughput vs. footprint (L2 hit/miss) and vs. the share
// of reductions that target one hot address (same-address serialisation).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/red_probe tools/red_probe.cu
//   tools/red_probe
//
// Each thread issues K reductions; address = hash(thread, k) within the
// footprint, except a `hot_ppm` share (parts per million) that go to one of
// `n_hot` hot words. Printed: G reductions/s.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}

__global__ void probe(uint32_t* buf, uint32_t words, uint32_t k_per_thread, uint32_t hot_ppm,
                      uint32_t n_hot) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    for (uint32_t k = 0; k < k_per_thread; ++k) {
        const uint32_t h = mix(tid * 0x9E3779B9u + k * 0x85EBCA6Bu);
        uint32_t a;
        if (h % 1000000u < hot_ppm) a = (h >> 8) % n_hot * 8191u % words; // hot words, spread
        else a = mix(h) % words;
        asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(buf + a), "r"(1u));
    }
}

int main() {
    uint32_t* buf;
    const size_t max_words = size_t(1) << 28; // 1 GiB
    cudaMalloc(&buf, max_words * 4);
    cudaMemset(buf, 0, max_words * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int block = 512, grid = 148 * 4;
    const uint32_t K = 256;
    const double total = double(block) * grid * K;
    auto run = [&](uint32_t words, uint32_t ppm, uint32_t n_hot, const char* tag) {
        probe<<<grid, block>>>(buf, words, K, ppm, n_hot);
        cudaEventRecord(a);
        for (int i = 0; i < 5; ++i) probe<<<grid, block>>>(buf, words, K, ppm, n_hot);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-28s footprint %8.2f MB  hot %6u ppm over %5u words: %7.2f G RED/s  (%.3f ms per 100M)\n",
               tag, words * 4.0 / 1e6, ppm, n_hot, total * 5 / (ms * 1e-3) / 1e9,
               100e6 / (total * 5 / (ms * 1e-3)) * 1e3);
    };
    for (uint32_t mb : {1u, 4u, 16u, 32u, 64u, 96u, 128u, 256u, 1024u})
        run(mb * (1u << 20) / 4, 0, 1, "footprint");
    for (uint32_t ppm : {10u, 100u, 500u, 1000u, 5000u})
        for (uint32_t nh : {1u, 16u, 256u})
            run(16u << 18, ppm, nh, "hot share (16 MB)");
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
