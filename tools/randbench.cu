// Random-access ceiling of the B200 memory system for the expansion's access pattern
// (DESIGN.md §6): 4-byte accesses at uniformly random word positions of a working set of
// `mb` MiB -- plain L2 loads (ld.global.cg), atomicAnd alone, and a load followed by a
// dependent atomicAnd on the same word (the relaxation's pattern) -- from a full grid with
// several independent chains per thread.  Prints one JSON line per (pattern, size).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o randbench tools/randbench.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t mix(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}
__device__ __forceinline__ uint64_t pick(uint64_t nwords, uint32_t t, uint32_t k) {
    const uint64_t r = (uint64_t)mix(t * 0x9E3779B9u + k) << 32 | mix(t ^ (k * 0x85EBCA6Bu) ^ 0x5bd1e995u);
    return r % nwords;
}

constexpr int CH = 4;  // independent chains per thread

template <int MODE> __device__ __forceinline__ uint32_t ld(const uint32_t *p) {
    uint32_t v;
    if (MODE == 3) v = *(volatile const uint32_t *)p;  // ld.volatile
    else if (MODE == 4) v = __ldg(p);                   // ld.global.nc
    else if (MODE == 5) v = __ldcs(p);                  // ld.global.cs (evict-first)
    else if (MODE == 6) v = __ldlu(p);                  // ld.global.lu
    else if (MODE == 7) v = __ldca(p);                  // ld.global.ca (L1)
    else if (MODE == 8) asm volatile("ld.global.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
    else if (MODE == 10 || MODE == 11) v = atomicOr((uint32_t *)p, 0u);  // atomic read at the home L2 slice
    else if (MODE == 12 || MODE == 13) {                // relaxed gpu-scope atomic load (ld.relaxed.gpu)
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
    } else if (MODE == 9) {                               // L2 evict_first cache policy
        uint64_t pol;
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("ld.global.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    } else v = __ldcg(p);
    return v;
}

// modes >= 20: load variant (MODE - 20) followed by the dependent atomicAnd
template <int MODE>  // 0 load, 1 atomicAnd, 2 load -> dependent atomicAnd, 3.. load variants (ld<MODE>)
__global__ void __launch_bounds__(256) k_rand(uint32_t *a, uint64_t nwords, int iters, uint32_t *sink) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t acc = 0;
    for (int it = 0; it < iters; it++) {
        uint64_t ix[CH];
        uint32_t v[CH];
#pragma unroll
        for (int c = 0; c < CH; c++) ix[c] = pick(nwords, t, it * CH + c);
        if (MODE == 0 || MODE >= 2) {
#pragma unroll
            for (int c = 0; c < CH; c++) v[c] = ld<(MODE >= 20 ? MODE - 20 : MODE)>(a + ix[c]);
        }
        if (MODE == 1) {
#pragma unroll
            for (int c = 0; c < CH; c++) v[c] = atomicAnd(a + ix[c], ~(1u << ((it + c) & 31)));
        }
        if (MODE == 2 || MODE == 11 || MODE == 13 || MODE >= 20) {
#pragma unroll
            for (int c = 0; c < CH; c++)
                if (v[c]) v[c] = atomicAnd(a + ix[c], ~(1u << ((it + c) & 31)));
        }
#pragma unroll
        for (int c = 0; c < CH; c++) acc += v[c];
    }
    if (acc == 0x12345678u) *sink = acc;
}

int main(int argc, char **argv) {
    const int iters = 64;
    size_t gran = 0;
    cudaDeviceGetLimit(&gran, cudaLimitMaxL2FetchGranularity);
    printf("{\"default_max_l2_fetch_granularity\": %zu}\n", gran);
    if (argc > 1) {  // cudaLimitMaxL2FetchGranularity (bytes) for this run
        cudaError_t e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, (size_t)atoi(argv[1]));
        cudaDeviceGetLimit(&gran, cudaLimitMaxL2FetchGranularity);
        printf("{\"set_max_l2_fetch_granularity\": %d, \"now\": %zu, \"err\": \"%s\"}\n", atoi(argv[1]), gran,
               cudaGetErrorString(e));
    }
    const unsigned blocks = 148 * 8, threads = 256;
    const uint64_t sizes_mb[] = {64, 8192};
    uint32_t *sink;
    cudaMalloc(&sink, 4);
    for (uint64_t mb : sizes_mb) {
        uint32_t *a = nullptr;
        const uint64_t bytes = mb << 20;
        if (cudaMalloc(&a, bytes) != cudaSuccess) { printf("{\"error\": \"malloc %llu MiB\"}\n", (unsigned long long)mb); return 1; }
        for (int mode = 0; mode < 30; mode++) {
            if (mode >= 14 && mode < 23) continue;
            cudaMemset(a, 0xFF, bytes);
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            float best = 1e30f;
            for (int rep = 0; rep < 5; rep++) {
                cudaEventRecord(e0);
                if (mode == 0) k_rand<0><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 1) k_rand<1><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 2) k_rand<2><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 3) k_rand<3><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 4) k_rand<4><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 5) k_rand<5><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 6) k_rand<6><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 7) k_rand<7><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 8) k_rand<8><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 9) k_rand<9><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 10) k_rand<10><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 11) k_rand<11><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 12) k_rand<12><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 13) k_rand<13><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 23) k_rand<23><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 24) k_rand<24><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 25) k_rand<25><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 26) k_rand<26><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 27) k_rand<27><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 28) k_rand<28><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                if (mode == 29) k_rand<29><<<blocks, threads>>>(a, bytes / 4, iters, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep > 0 && ms < best) best = ms;  // first launch is a warm-up
            }
            cudaError_t err = cudaGetLastError();
            const double acc = (double)blocks * threads * iters * CH * (mode == 2 || mode == 11 || mode == 13 || mode >= 20 ? 2 : 1);
            const char *name[] = {"load.cg", "atomicAnd", "load.cg+atomicAnd", "load.volatile", "load.nc", "load.cs",
                                  "load.lu", "load.ca", "load.L1::no_allocate", "load.L2::evict_first",
                                  "atomicOr0", "atomicOr0+atomicAnd", "ld.relaxed.gpu", "ld.relaxed.gpu+atomicAnd",
                                  "", "", "", "", "", "", "", "", "", "load.volatile+atomicAnd", "load.nc+atomicAnd",
                                  "load.cs+atomicAnd", "load.lu+atomicAnd", "load.ca+atomicAnd",
                                  "load.L1::no_allocate+atomicAnd", "load.L2::evict_first+atomicAnd"};
            printf("{\"pattern\": \"%s\", \"working_set_mib\": %llu, \"ms\": %.3f, \"g_accesses_per_s\": %.2f, "
                   "\"gb_s_at_32B\": %.0f, \"gb_s_at_64B\": %.0f, \"err\": \"%s\"}\n",
                   name[mode], (unsigned long long)mb, best, acc / best / 1e6, acc * 32 / best / 1e6,
                   acc * 64 / best / 1e6, cudaGetErrorString(err));
            fflush(stdout);
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
        }
        cudaFree(a);
    }
    return 0;
}
