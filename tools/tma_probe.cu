// tma_probe.cu — microbenchmark: streaming 6 SoA columns (32 B/record) with
// (a) direct 128-bit loads, (b) the K2 TMA pipeline with trivial consumers.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_probe tools/tma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr uint32_t kTile = 1024, kStages = 3, kChunks = kTile / 32, kStageBytes = kTile * 32;

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}" ::"r"(su(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void tma(void* d, const void* s, uint32_t n, uint64_t* b, uint64_t pol) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 ::"r"(su(d)), "l"(s), "r"(n), "r"(su(b)), "l"(pol) : "memory");
}
__device__ __forceinline__ void tma_nohint(void* d, const void* s, uint32_t n, uint64_t* b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(su(d)), "l"(s), "r"(n), "r"(su(b)) : "memory");
}

struct Cols { const uint32_t *a, *b, *c, *d; const uint64_t *e, *f; uint64_t n; };

__global__ void direct(Cols c, unsigned long long* out) {
    uint64_t acc = 0;
    const uint64_t n4 = c.n / 4, stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < n4; g += stride) {
        uint4 x = __ldcs((const uint4*)c.a + g), y = __ldcs((const uint4*)c.b + g), z = __ldcs((const uint4*)c.c + g), w = __ldcs((const uint4*)c.d + g);
        ulonglong2 e0 = __ldcs((const ulonglong2*)c.e + 2 * g), e1 = __ldcs((const ulonglong2*)c.e + 2 * g + 1);
        ulonglong2 f0 = __ldcs((const ulonglong2*)c.f + 2 * g), f1 = __ldcs((const ulonglong2*)c.f + 2 * g + 1);
        acc += x.x + y.y + z.z + w.w + e0.x + e1.y + f0.x + f1.y;
    }
    if (acc == 42) *out = acc;
}

// mode 0: dynamic claim; 1: static chunk assignment; bit 2 (4): no L2 hint
__global__ void __launch_bounds__(1024, 1) piped(Cols c, unsigned long long* out, int mode) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t* full = (uint64_t*)(sm + kStages * kStageBytes);
    uint64_t* empty = full + kStages;
    uint32_t* claim = (uint32_t*)(empty + kStages);
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t nv = c.n & ~3ull, nt = (nv + kTile - 1) / kTile;
    const uint32_t my = blockIdx.x < nt ? (uint32_t)((nt - blockIdx.x + gridDim.x - 1) / gridDim.x) : 0;
    if (threadIdx.x == 0) {
        for (uint32_t s = 0; s < kStages; ++s) { mbar_init(full + s, 1); mbar_init(empty + s, kChunks); }
        *claim = 0;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint64_t acc = 0;
    if (warp == 0) {
        if (lane == 0) {
            uint64_t pol;
            asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
            for (uint32_t j = 0; j < my; ++j) {
                const uint32_t s = j % kStages;
                if (j >= kStages) mbar_wait(empty + s, ((j / kStages) - 1) & 1);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                const uint64_t f = ((uint64_t)blockIdx.x + (uint64_t)j * gridDim.x) * kTile;
                const uint32_t cnt = (uint32_t)min((uint64_t)kTile, nv - f);
                unsigned char* st = sm + s * kStageBytes;
                mbar_expect(full + s, cnt * 32);
                if (mode & 4) {
                    tma_nohint(st, c.a + f, cnt * 4, full + s); tma_nohint(st + 4096, c.b + f, cnt * 4, full + s);
                    tma_nohint(st + 8192, c.c + f, cnt * 4, full + s); tma_nohint(st + 12288, c.d + f, cnt * 4, full + s);
                    tma_nohint(st + 16384, c.e + f, cnt * 8, full + s); tma_nohint(st + 24576, c.f + f, cnt * 8, full + s);
                } else {
                    tma(st, c.a + f, cnt * 4, full + s, pol); tma(st + 4096, c.b + f, cnt * 4, full + s, pol);
                    tma(st + 8192, c.c + f, cnt * 4, full + s, pol); tma(st + 12288, c.d + f, cnt * 4, full + s, pol);
                    tma(st + 16384, c.e + f, cnt * 8, full + s, pol); tma(st + 24576, c.f + f, cnt * 8, full + s, pol);
                }
            }
        }
        __syncwarp();
    } else {
        const uint32_t nw = (blockDim.x >> 5) - 1;
        for (uint32_t it = 0;; ++it) {
            uint32_t cl;
            if ((mode & 3) == 0) {
                cl = 0;
                if (lane == 0) cl = atomicAdd(claim, 1u);
                cl = __shfl_sync(~0u, cl, 0);
            } else {
                cl = (warp - 1) + it * nw;
            }
            if (cl >= my * kChunks) break;
            const uint32_t i = cl / kChunks, ch = cl % kChunks, s = i % kStages;
            mbar_wait(full + s, (i / kStages) & 1);
            const unsigned char* st = sm + s * kStageBytes;
            const uint32_t k = ch * 32 + lane;
            acc += ((const uint32_t*)st)[k] + ((const uint32_t*)(st + 4096))[k] + ((const uint32_t*)(st + 8192))[k] +
                   ((const uint32_t*)(st + 12288))[k] + ((const uint64_t*)(st + 16384))[k] + ((const uint64_t*)(st + 24576))[k];
            __syncwarp();
            if (lane == 0) mbar_arrive(empty + s);
        }
    }
    if (acc == 42) *out = acc;
}

int main() {
    const uint64_t n = 100000000;
    Cols c;
    void* p;
    cudaMalloc(&p, n * 32);
    cudaMemset(p, 1, n * 32);
    unsigned char* b = (unsigned char*)p;
    c.a = (uint32_t*)b; c.b = (uint32_t*)(b + n * 4); c.c = (uint32_t*)(b + n * 8); c.d = (uint32_t*)(b + n * 12);
    c.e = (uint64_t*)(b + n * 16); c.f = (uint64_t*)(b + n * 24); c.n = n;
    unsigned long long* out;
    cudaMalloc(&out, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t smem = kStages * kStageBytes + 64;
    cudaFuncSetAttribute(piped, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto run = [&](const char* name, auto launch) {
        for (int i = 0; i < 3; ++i) launch();
        cudaEventRecord(e0);
        for (int i = 0; i < 10; ++i) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 10;
        printf("%-28s %8.3f ms  %8.1f GB/s  err=%s\n", name, ms, n * 32 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    run("direct 296x512", [&] { direct<<<sms * 2, 512>>>(c, out); });
    run("direct 148x1024", [&] { direct<<<sms, 1024>>>(c, out); });
    run("direct 592x512", [&] { direct<<<sms * 4, 512>>>(c, out); });
    run("tma dynamic claim", [&] { piped<<<sms, 1024, smem>>>(c, out, 0); });
    run("tma static", [&] { piped<<<sms, 1024, smem>>>(c, out, 1); });
    run("tma dynamic, no L2 hint", [&] { piped<<<sms, 1024, smem>>>(c, out, 4); });
    run("tma static, no L2 hint", [&] { piped<<<sms, 1024, smem>>>(c, out, 5); });
    return 0;
}
