// hops.cu -- Abar estimation by sampled shortest hop distances.
//
// Eq. 1-3 scale the fine weights around Abar, "the average shortest hops in the
// graph", which the paper estimates from "ten thousand pairs of nodes".  The
// caller draws the pairs; this computes every pair's hop distance (fewest edges of a directed
// path in the caller's edge list -- bidirected, so the undirected distance) with batched,
// level-synchronous BFS on the device: one BFS per distinct source, B sources in flight, a
// visited bitmap per source (test-and-set by atomicOr: the first visitor appends the node to
// the source's next queue), one warp per frontier node with the lanes over its out-row (hubs
// do not serialise a thread), and early exit of a source once all its targets are reached.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "internal.cuh"

namespace {

constexpr uint32_t HOP_INF = 0xFFFFFFFFu;

struct BfsDev {
    uint32_t V, W, B;
    uint32_t *vis;               // [B][W] visited bitmaps
    uint32_t *q[2];              // [B][V] frontier queues (a node enters a source's queue once)
    uint32_t *qn[2];             // [B] queue sizes
    unsigned long long *offs;    // [B + 1] prefix of the current queue sizes
    uint32_t *pb, *pt, *pd;      // pairs of this batch: source slot, target (internal id), distance
    uint32_t np;
    uint32_t *unres;             // [B] unresolved pairs per source slot
};

__global__ void k_bfs_seed(BfsDev d, const uint32_t *srcs, uint32_t nb) {
    for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x) {
        const uint32_t s = srcs[b];
        d.vis[(size_t)b * d.W + (s >> 5)] |= 1u << (s & 31);
        d.q[0][(size_t)b * d.V] = s;
        d.qn[0][b] = 1;
    }
}

// after level L's expansion (or the seed, L = 0 with `level` = 0): pairs whose target is now
// visited get d = level; count the unresolved pairs per source
__global__ void k_bfs_resolve(BfsDev d, uint32_t level) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < d.np; i += gridDim.x * blockDim.x) {
        if (d.pd[i] != HOP_INF) continue;
        const uint32_t b = d.pb[i], t = d.pt[i];
        if ((d.vis[(size_t)b * d.W + (t >> 5)] >> (t & 31)) & 1u) d.pd[i] = level;
        else atomicAdd(&d.unres[b], 1u);
    }
}

// one block: drop the queues of finished sources, prefix of the remaining queue sizes
__global__ void k_bfs_plan(BfsDev d, uint32_t cur, uint32_t nb, uint32_t *total_out) {
    __shared__ unsigned long long sc[1024];
    const uint32_t b = threadIdx.x;
    unsigned long long n = 0;
    if (b < nb) {
        n = d.unres[b] ? d.qn[cur][b] : 0;  // every target of this source found: stop its BFS
        d.qn[cur ^ 1][b] = 0;
        d.unres[b] = 0;
    }
    sc[b] = n;
    __syncthreads();
    for (uint32_t o = 1; o < 1024; o <<= 1) {
        unsigned long long v = b >= o ? sc[b - o] : 0;
        __syncthreads();
        sc[b] += v;
        __syncthreads();
    }
    if (b < nb) d.offs[b] = sc[b] - n;
    if (b == 0) {
        d.offs[nb] = sc[1023];
        *total_out = (uint32_t)min(sc[1023], 0xFFFFFFFFull);
    }
}

__global__ void __launch_bounds__(256) k_bfs_expand(GraphDev g, BfsDev d, uint32_t cur, uint32_t nb) {
    const uint32_t lane = threadIdx.x & 31;
    const unsigned long long total = d.offs[nb];
    const unsigned long long w0 = (blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nw = (gridDim.x * (unsigned long long)blockDim.x) >> 5;
    for (unsigned long long base = w0 * 32; base < total; base += nw * 32) {
        // item of this lane: (source slot b, queue position)
        const unsigned long long item = base + lane;
        uint32_t b = 0, f = 0;
        bool valid = item < total;
        if (valid) {
            uint32_t lo = 0, hi = nb;  // largest b with offs[b] <= item
            while (hi - lo > 1) {
                const uint32_t m = (lo + hi) >> 1;
                if (d.offs[m] <= item) lo = m; else hi = m;
            }
            b = lo;
            f = d.q[cur][(size_t)b * d.V + (uint32_t)(item - d.offs[b])];
        }
        unsigned vm = __ballot_sync(0xFFFFFFFFu, valid);
        while (vm) {  // the warp walks each item's out-row, lanes over the edges
            const int src = __ffs(vm) - 1;
            vm &= vm - 1;
            const uint32_t bb = __shfl_sync(0xFFFFFFFFu, b, src), ff = __shfl_sync(0xFFFFFFFFu, f, src);
            const uint32_t rb = __ldg(g.row + ff), re = __ldg(g.row + ff + 1);
            uint32_t *vis = d.vis + (size_t)bb * d.W;
            for (uint32_t k0 = rb; k0 < re; k0 += 32) {
                const uint32_t k = k0 + lane;
                bool add = false;
                uint32_t n = 0;
                if (k < re) {
                    n = __ldg(g.col + k);
                    const uint32_t bit = 1u << (n & 31);
                    if (!(__ldcg(vis + (n >> 5)) & bit)) add = !(atomicOr(vis + (n >> 5), bit) & bit);
                }
                const unsigned am = __ballot_sync(0xFFFFFFFFu, add);
                if (am) {
                    uint32_t pos = 0;
                    if (lane == 0) pos = atomicAdd(&d.qn[cur ^ 1][bb], (uint32_t)__popc(am));
                    pos = __shfl_sync(0xFFFFFFFFu, pos, 0);
                    if (add) d.q[cur ^ 1][(size_t)bb * d.V + pos + __popc(am & ((1u << lane) - 1))] = n;
                }
            }
        }
    }
}

// plain out-CSR (internal ids) for a graph whose activation-sorted CSR is not built yet
__global__ void k_src_keys(const uint32_t *src, uint64_t E, unsigned long long *keys, uint32_t *deg) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < E; e += (uint64_t)gridDim.x * blockDim.x) {
        keys[e] = (unsigned long long)src[e] << 32 | e;
        atomicAdd(&deg[src[e]], 1u);
    }
}
__global__ void k_gather_col(const unsigned long long *keys, const uint32_t *dst, uint64_t E, uint32_t *col) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < E; i += (uint64_t)gridDim.x * blockDim.x)
        col[i] = dst[(uint32_t)keys[i]];
}

__global__ void k_to_internal(const uint32_t *perm, const uint32_t *in, uint32_t n, uint32_t *out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = perm[in[i]];
}

}  // namespace

void graph_sample_hops(riki_graph *g, uint32_t n_pairs, const uint32_t *src, const uint32_t *dst, uint32_t max_hops,
                       uint32_t *dist_out) {
    for (uint32_t i = 0; i < n_pairs; i++)
        if (src[i] >= g->V || dst[i] >= g->V) RIKI_THROW(RIKI_EINVAL, "pair node out of range");
    cudaStream_t s = g->stream;
    const uint32_t V = g->V, W = (V + 31) / 32;
    GraphDev gd = g->dev();
    uint32_t *t_row = nullptr, *t_col = nullptr;  // plain CSR when no activation levels are set yet
    struct Tmp {
        std::vector<void *> p;
        ~Tmp() { for (void *x : p) cudaFree(x); }
    } tmp_csr;
    if (!g->has_act) {
        const uint64_t E = g->E;
        unsigned long long *k1 = nullptr, *k2 = nullptr;
        CUDA_TRY(cudaMalloc(&t_row, (V + 1) * 4ull)); tmp_csr.p.push_back(t_row);
        CUDA_TRY(cudaMalloc(&t_col, std::max<uint64_t>(E, 1) * 4)); tmp_csr.p.push_back(t_col);
        CUDA_TRY(cudaMalloc(&k1, std::max<uint64_t>(E, 1) * 8)); tmp_csr.p.push_back(k1);
        CUDA_TRY(cudaMalloc(&k2, std::max<uint64_t>(E, 1) * 8)); tmp_csr.p.push_back(k2);
        CUDA_TRY(cudaMemsetAsync(t_row, 0, (V + 1) * 4ull, s));
        if (E) {
            k_src_keys<<<1184, 256, 0, s>>>(g->d_src, E, k1, t_row);
            size_t tb = 0, tb2 = 0;
            CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tb, k1, k2, (int64_t)E, 0, 64, s));
            CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb2, t_row, t_row, (int64_t)V + 1, s));
            void *tbuf = nullptr;
            CUDA_TRY(cudaMalloc(&tbuf, std::max(tb, tb2))); tmp_csr.p.push_back(tbuf);
            size_t t1 = std::max(tb, tb2);
            CUDA_TRY(cub::DeviceRadixSort::SortKeys(tbuf, t1, k1, k2, (int64_t)E, 0, 64, s));
            t1 = std::max(tb, tb2);
            CUDA_TRY(cub::DeviceScan::ExclusiveSum(tbuf, t1, t_row, t_row, (int64_t)V + 1, s));
            k_gather_col<<<1184, 256, 0, s>>>(k2, g->d_dst, E, t_col);
        }
        gd.row = t_row;
        gd.col = t_col;
    }
    // group the pairs by source (caller ids); B distinct sources in flight per batch
    std::vector<uint32_t> order(n_pairs);
    std::iota(order.begin(), order.end(), 0u);
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return src[a] < src[b]; });
    size_t fr = 0, tot = 0;
    CUDA_TRY(cudaMemGetInfo(&fr, &tot));
    const uint64_t per_src = (uint64_t)W * 4 + 2ull * V * 4 + 64;
    const uint64_t budget = fr > (4ull << 30) ? (fr - (4ull << 30)) / 2 : fr / 4;
    const uint32_t B = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(1024, budget / per_src));
    BfsDev d{};
    d.V = V; d.W = W; d.B = B;
    uint32_t *pool = nullptr;
    const size_t words = (size_t)B * W + 2 * (size_t)B * V + 2 * (size_t)B + B;
    CUDA_TRY(cudaMalloc(&pool, words * 4));
    unsigned long long *offs = nullptr;
    uint32_t *pairs = nullptr, *total_d = nullptr, *srcs = nullptr, *tmp = nullptr;
    uint32_t *h_total = nullptr;
    try {
        CUDA_TRY(cudaMalloc(&offs, (B + 1) * 8));
        CUDA_TRY(cudaMalloc(&pairs, 3ull * std::max<uint32_t>(n_pairs, 1) * 4));
        CUDA_TRY(cudaMalloc(&srcs, (size_t)B * 4));
        CUDA_TRY(cudaMalloc(&tmp, (size_t)std::max<uint32_t>(n_pairs, B) * 4));
        CUDA_TRY(cudaMalloc(&total_d, 4));
        CUDA_TRY(cudaMallocHost(&h_total, 4));
        d.vis = pool;
        d.q[0] = pool + (size_t)B * W;
        d.q[1] = d.q[0] + (size_t)B * V;
        d.qn[0] = d.q[1] + (size_t)B * V;
        d.qn[1] = d.qn[0] + B;
        d.unres = d.qn[1] + B;
        d.offs = offs;
        for (uint32_t i0 = 0; i0 < n_pairs;) {
            // next batch: pairs of up to B distinct sources
            std::vector<uint32_t> bsrc, pb, pt, idx;
            uint32_t i = i0;
            while (i < n_pairs) {
                const uint32_t sv = src[order[i]];
                if (bsrc.empty() || bsrc.back() != sv) {
                    if (bsrc.size() == B) break;
                    bsrc.push_back(sv);
                }
                pb.push_back((uint32_t)bsrc.size() - 1);
                pt.push_back(dst[order[i]]);
                idx.push_back(order[i]);
                i++;
            }
            const uint32_t nb = (uint32_t)bsrc.size(), np = i - i0;
            i0 = i;
            d.pb = pairs; d.pt = pairs + np; d.pd = pairs + 2 * np; d.np = np;
            CUDA_TRY(cudaMemcpyAsync(d.pb, pb.data(), np * 4, cudaMemcpyHostToDevice, s));
            CUDA_TRY(cudaMemcpyAsync(tmp, pt.data(), np * 4, cudaMemcpyHostToDevice, s));
            k_to_internal<<<(np + 255) / 256, 256, 0, s>>>(g->d_perm, tmp, np, d.pt);
            CUDA_TRY(cudaMemcpyAsync(tmp, bsrc.data(), nb * 4, cudaMemcpyHostToDevice, s));
            k_to_internal<<<(nb + 255) / 256, 256, 0, s>>>(g->d_perm, tmp, nb, srcs);
            CUDA_TRY(cudaMemsetAsync(d.pd, 0xFF, np * 4, s));
            CUDA_TRY(cudaMemsetAsync(d.vis, 0, (size_t)nb * W * 4, s));
            CUDA_TRY(cudaMemsetAsync(d.qn[0], 0, 3ull * B * 4, s));  // qn[0], qn[1], unres
            k_bfs_seed<<<(nb + 255) / 256, 256, 0, s>>>(d, srcs, nb);
            k_bfs_resolve<<<std::min<uint32_t>((np + 255) / 256, 1184), 256, 0, s>>>(d, 0);
            uint32_t cur = 0;
            for (uint32_t level = 0; level < max_hops; level++) {
                k_bfs_plan<<<1, 1024, 0, s>>>(d, cur, nb, total_d);
                CUDA_TRY(cudaMemcpyAsync(h_total, total_d, 4, cudaMemcpyDeviceToHost, s));
                CUDA_TRY(cudaStreamSynchronize(s));
                if (*h_total == 0) break;
                k_bfs_expand<<<148 * 8, 256, 0, s>>>(gd, d, cur, nb);
                k_bfs_resolve<<<std::min<uint32_t>((np + 255) / 256, 1184), 256, 0, s>>>(d, level + 1);
                CUDA_TRY(cudaGetLastError());
                cur ^= 1;
            }
            std::vector<uint32_t> dist(np);
            CUDA_TRY(cudaMemcpyAsync(dist.data(), d.pd, np * 4, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            for (uint32_t j = 0; j < np; j++) dist_out[idx[j]] = dist[j];
        }
    } catch (...) {
        cudaFree(pool); cudaFree(offs); cudaFree(pairs); cudaFree(srcs); cudaFree(tmp); cudaFree(total_d);
        if (h_total) cudaFreeHost(h_total);
        throw;
    }
    cudaFree(pool); cudaFree(offs); cudaFree(pairs); cudaFree(srcs); cudaFree(tmp); cudaFree(total_d);
    cudaFreeHost(h_total);
}
