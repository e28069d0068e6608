// common.cuh -- internal helpers of libriki.so (sm_100a).  Not part of the C-ABI.
// Byte-SIMD row arithmetic for the node-keyword matrix H, warp utilities,
// CTA-scope hash sets and sorts used by the recovery kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#define RIKI_INF 0xFFu
#define WARP 32
#define FULLMASK 0xffffffffu

// ------------------------------------------------------------------ byte-SIMD rows
// An H row is one machine word holding up to 4 (uint32_t) or 8 (uint64_t) one-byte
// hitting levels, node-major.  Unused bytes are kept at 0 so that "no 0xFF byte" means
// "row complete" and "all bytes <= l" means "blocked at level l" (R10 closed form).
template <class W> struct Row;

template <> struct Row<uint32_t> {
    static constexpr int BYTES = 4;
    __device__ __forceinline__ static uint32_t splat(uint32_t b) { return b * 0x01010101u; }
    __device__ __forceinline__ static uint32_t eq(uint32_t x, uint32_t y) { return __vcmpeq4(x, y); }
    __device__ __forceinline__ static uint32_t lt(uint32_t x, uint32_t y) { return __vcmpltu4(x, y); }
    __device__ __forceinline__ static uint32_t le(uint32_t x, uint32_t y) { return __vcmpleu4(x, y); }
    __device__ __forceinline__ static uint32_t maxb(uint32_t x) {  // max byte
        uint32_t m = __vmaxu4(x, x >> 16);
        m = __vmaxu4(m, m >> 8);
        return m & 0xFF;
    }
    __device__ __forceinline__ static int ones(uint32_t m) { return __popc(m) >> 3; }  // # selected bytes
    __device__ __forceinline__ static uint32_t byte(uint32_t x, int j) { return (x >> (8 * j)) & 0xFF; }
    __device__ __forceinline__ static uint32_t atomic_and(uint32_t *p, uint32_t m) { return atomicAnd(p, m); }
    __device__ __forceinline__ static uint32_t load(const uint32_t *p) { return __ldcg(p); }
};

// 16-bit rows (<= 2 keywords): computed as the low half of a 32-bit SIMD word (upper bytes 0);
// the atomic goes through the containing aligned 32-bit word with the other half kept by 0xFFFF.
template <> struct Row<uint16_t> {
    static constexpr int BYTES = 2;
    __device__ __forceinline__ static uint16_t splat(uint32_t b) { return (uint16_t)(b * 0x0101u); }
    __device__ __forceinline__ static uint16_t eq(uint32_t x, uint32_t y) { return (uint16_t)__vcmpeq4(x, y); }
    __device__ __forceinline__ static uint16_t lt(uint32_t x, uint32_t y) { return (uint16_t)__vcmpltu4(x, y); }
    __device__ __forceinline__ static uint16_t le(uint32_t x, uint32_t y) { return (uint16_t)__vcmpleu4(x, y); }
    __device__ __forceinline__ static uint32_t maxb(uint32_t x) { return max(x & 0xFFu, (x >> 8) & 0xFFu); }
    __device__ __forceinline__ static int ones(uint32_t m) { return __popc(m & 0xFFFFu) >> 3; }
    __device__ __forceinline__ static uint32_t byte(uint32_t x, int j) { return (x >> (8 * j)) & 0xFF; }
    __device__ __forceinline__ static uint16_t atomic_and(uint16_t *p, uint32_t m) {
        uintptr_t a = (uintptr_t)p;
        uint32_t sh = (uint32_t)(a & 2) * 8;
        uint32_t m32 = ((m & 0xFFFFu) << sh) | (0xFFFFu << (16 - sh));
        uint32_t old = atomicAnd((uint32_t *)(a & ~(uintptr_t)3), m32);
        return (uint16_t)(old >> sh);
    }
    __device__ __forceinline__ static uint16_t load(const uint16_t *p) { return __ldcg((const unsigned short *)p); }
};

template <> struct Row<uint64_t> {
    static constexpr int BYTES = 8;
    __device__ __forceinline__ static uint64_t pack(uint32_t lo, uint32_t hi) { return (uint64_t)hi << 32 | lo; }
    __device__ __forceinline__ static uint64_t splat(uint32_t b) { return (uint64_t)b * 0x0101010101010101ull; }
    __device__ __forceinline__ static uint64_t eq(uint64_t x, uint64_t y) {
        return pack(__vcmpeq4((uint32_t)x, (uint32_t)y), __vcmpeq4((uint32_t)(x >> 32), (uint32_t)(y >> 32)));
    }
    __device__ __forceinline__ static uint64_t lt(uint64_t x, uint64_t y) {
        return pack(__vcmpltu4((uint32_t)x, (uint32_t)y), __vcmpltu4((uint32_t)(x >> 32), (uint32_t)(y >> 32)));
    }
    __device__ __forceinline__ static uint64_t le(uint64_t x, uint64_t y) {
        return pack(__vcmpleu4((uint32_t)x, (uint32_t)y), __vcmpleu4((uint32_t)(x >> 32), (uint32_t)(y >> 32)));
    }
    __device__ __forceinline__ static uint32_t maxb(uint64_t x) {
        uint32_t m = __vmaxu4((uint32_t)x, (uint32_t)(x >> 32));
        m = __vmaxu4(m, m >> 16);
        m = __vmaxu4(m, m >> 8);
        return m & 0xFF;
    }
    __device__ __forceinline__ static int ones(uint64_t m) { return __popcll(m) >> 3; }
    __device__ __forceinline__ static uint32_t byte(uint64_t x, int j) { return (uint32_t)(x >> (8 * j)) & 0xFF; }
    __device__ __forceinline__ static uint64_t atomic_and(uint64_t *p, uint64_t m) {
        return atomicAnd((unsigned long long *)p, (unsigned long long)m);
    }
    __device__ __forceinline__ static uint64_t load(const uint64_t *p) {
        return __ldcg((const unsigned long long *)p);
    }
};

// ------------------------------------------------------------------ warp helpers
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}
template <class T> __device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T n = __shfl_up_sync(FULLMASK, v, o);
        if ((int)lane_id() >= o) v += n;
    }
    return v;
}
template <class T> __device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
    return v;
}

// Warp-aggregated append of `val` to list[*counter] grouped by `key` (lanes with want).
// Must be called by all 32 lanes (convergent).  Returns the slot index or UINT32_MAX.
__device__ __forceinline__ uint32_t warp_append(bool want, uint32_t key, uint32_t *counter_base,
                                                uint32_t counter_stride) {
    uint32_t m = __ballot_sync(FULLMASK, want);
    uint32_t pos = UINT32_MAX;
    if (want) {
        uint32_t peers = __match_any_sync(m, key);
        uint32_t leader = __ffs(peers) - 1;
        uint32_t rank = __popc(peers & lanemask_lt());
        uint32_t base = 0;
        if (lane_id() == leader) base = atomicAdd(counter_base + (size_t)key * counter_stride, __popc(peers));
        base = __shfl_sync(peers, base, leader);
        pos = base + rank;
    }
    return pos;
}

// ------------------------------------------------------------------ CTA hash set (node ids)
// Open addressing, linear probing, EMPTY = 0xFFFFFFFF, capacity a power of two.  Lives in
// shared memory (fast path) or global scratch (overflow path); same code.
struct HashSet {
    uint32_t *keys;
    uint32_t cap;  // power of two
    __device__ __forceinline__ static uint32_t hash(uint32_t x) {
        x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
        return x;
    }
    // returns 1 = inserted, 0 = present, -1 = full
    __device__ __forceinline__ int insert(uint32_t k, uint32_t *slot_out = nullptr) const {
        uint32_t h = hash(k) & (cap - 1);
        for (uint32_t i = 0; i < cap; i++) {
            uint32_t s = (h + i) & (cap - 1);
            uint32_t prev = atomicCAS(&keys[s], 0xFFFFFFFFu, k);
            if (prev == 0xFFFFFFFFu) { if (slot_out) *slot_out = s; return 1; }
            if (prev == k) { if (slot_out) *slot_out = s; return 0; }
        }
        return -1;
    }
    __device__ __forceinline__ int find(uint32_t k) const {
        uint32_t h = hash(k) & (cap - 1);
        for (uint32_t i = 0; i < cap; i++) {
            uint32_t s = (h + i) & (cap - 1);
            uint32_t v = keys[s];
            if (v == k) return (int)s;
            if (v == 0xFFFFFFFFu) return -1;
        }
        return -1;
    }
};

// ------------------------------------------------------------------ CTA bitonic sort
// Sorts n keys ascending in place (keys in shared or global memory).  The buffer must hold
// next_pow2(n) entries: slots [n, N) are filled with the maximum key and end up at the tail.
__host__ __device__ __forceinline__ uint32_t next_pow2(uint32_t n) {
    uint32_t N = 1;
    while (N < n) N <<= 1;
    return N;
}
template <class K> __device__ void cta_bitonic_sort(K *keys, uint32_t n) {
    if (n < 2) return;
    const uint32_t N = next_pow2(n);
    const K KMAX = (K)~(K)0;
    for (uint32_t i = n + threadIdx.x; i < N; i += blockDim.x) keys[i] = KMAX;
    __syncthreads();
    for (uint32_t k = 2; k <= N; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
                uint32_t ixj = i ^ j;
                if (ixj > i) {
                    K a = keys[i], b = keys[ixj];
                    bool up = (i & k) == 0;
                    if ((a > b) == up) { keys[i] = b; keys[ixj] = a; }
                }
            }
            __syncthreads();
        }
    }
}

// ------------------------------------------------------------------ error plumbing
struct RikiError {
    int code;
    std::string msg;
};

#define CUDA_TRY(x)                                                                                   \
    do {                                                                                              \
        cudaError_t _e = (x);                                                                         \
        if (_e != cudaSuccess) {                                                                      \
            throw RikiError{-3, std::string(#x) + ": " + cudaGetErrorString(_e)};                     \
        }                                                                                             \
    } while (0)

#define RIKI_THROW(code, msg) throw RikiError{code, msg}
