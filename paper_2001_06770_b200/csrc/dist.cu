// dist.cu -- multi-GPU plumbing of libriki.so.
//
// Replicated mode (0) needs nothing here: queries are independent units, each rank runs its
// shard of a batch on its own replica and the host gathers the (small) result sets.
//
// Vertex-partitioned mode (1): the per-level exchange of the frontier bit-planes, one
// in-place ncclAllGather on the search stream (NCCL has no bitwise-OR reduction, so the
// exchange is owner-computes + all-gather).  NCCL is resolved at run time with
// dlopen (the copy torch already loaded if there is one, RTLD_NOLOAD first), so libriki.so
// has no link-time NCCL dependency and single-GPU use never touches it.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>

#include "internal.cuh"

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_gather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char *(*error_string)(ncclResult_t) = nullptr;
};

const NcclApi &nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) {
        if (!api.all_gather) RIKI_THROW(RIKI_ENCCL, "NCCL (libnccl.so.2) could not be loaded");
        return api;
    }
    tried = true;
    void *h = nullptr;
    if (const char *p = getenv("RIKI_NCCL_LIB")) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // torch's copy, if loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) RIKI_THROW(RIKI_ENCCL, std::string("dlopen libnccl.so.2: ") + dlerror());
    api.get_unique_id = (decltype(api.get_unique_id))dlsym(h, "ncclGetUniqueId");
    api.comm_init_rank = (decltype(api.comm_init_rank))dlsym(h, "ncclCommInitRank");
    api.all_gather = (decltype(api.all_gather))dlsym(h, "ncclAllGather");
    api.all_reduce = (decltype(api.all_reduce))dlsym(h, "ncclAllReduce");
    api.comm_destroy = (decltype(api.comm_destroy))dlsym(h, "ncclCommDestroy");
    api.error_string = (decltype(api.error_string))dlsym(h, "ncclGetErrorString");
    if (!api.get_unique_id || !api.comm_init_rank || !api.all_gather || !api.all_reduce || !api.comm_destroy ||
        !api.error_string) {
        api.all_gather = nullptr;
        RIKI_THROW(RIKI_ENCCL, "libnccl.so.2 lacks a required symbol");
    }
    return api;
}

void nccl_try(ncclResult_t r, const char *what) {
    if (r != ncclSuccess) RIKI_THROW(RIKI_ENCCL, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

void dist_unique_id(void *out128) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    nccl_try(nccl().get_unique_id(&id), "ncclGetUniqueId");
    memcpy(out128, &id, sizeof(id));
}

// Contiguous internal-id ranges balanced by pull work: a level scans every owned node's
// row (1) and up to its whole in-row (in-degree), so node v weighs indeg(v) + 1.  Internal
// ids are degree-descending, so the first ranges are short runs of hubs.  Every bound is a
// multiple of 32 or V (one bit-plane word never straddles two ranks); ranges may be empty
// when V is small.
void dist_partition(const uint32_t *irow, uint32_t V, uint32_t P, uint32_t *bounds) {
    const uint64_t total = (uint64_t)irow[V] + V;
    bounds[0] = 0;
    uint32_t v = 0;
    for (uint32_t r = 1; r < P; r++) {
        const uint64_t target = (total * r + P - 1) / P;  // ceil(total * r / P)
        // first 32-aligned v with weight(prefix [0, v)) >= target
        uint32_t lo = v, hi = V;
        while (lo < hi) {
            uint32_t m = lo + (hi - lo) / 2;
            if ((uint64_t)irow[m] + m >= target) hi = m; else lo = m + 1;
        }
        const uint32_t b = (uint32_t)std::min<uint64_t>(((uint64_t)lo + 31) / 32 * 32, V);  // >= bounds[r-1]
        bounds[r] = b;
        v = b;
    }
    bounds[P] = V;
}

void dist_init(riki_graph *g, int nranks, int rank, const void *uid, int mode) {
    if (nranks < 1 || nranks > 1024) RIKI_THROW(RIKI_EINVAL, "nranks must be in [1, 1024]");
    if (rank < 0 || rank >= nranks) RIKI_THROW(RIKI_EINVAL, "rank out of range");
    if (mode != 0 && mode != 1) RIKI_THROW(RIKI_EINVAL, "mode must be 0 (replicated) or 1 (vertex-partitioned)");
    dist_free(g);
    DistState *d = new DistState();
    d->nranks = nranks;
    d->rank = rank;
    d->mode = mode;
    d->push = getenv("RIKI_VP_PULL") == nullptr;  // push (fused exchange) unless the pull variant is asked for
    try {
        if (mode == 1) {
            d->simulated = uid == nullptr && nranks > 1;
            if (uid == nullptr && !d->simulated && nranks > 1) RIKI_THROW(RIKI_EINVAL, "missing NCCL unique id");
            std::vector<uint32_t> irow(g->V + 1);
            CUDA_TRY(cudaMemcpy(irow.data(), g->d_irow, (g->V + 1) * 4, cudaMemcpyDeviceToHost));
            d->bounds.resize(nranks + 1);
            dist_partition(irow.data(), g->V, nranks, d->bounds.data());
            uint32_t maxn = 0;
            for (int r = 0; r < nranks; r++) maxn = std::max(maxn, d->bounds[r + 1] - d->bounds[r]);
            d->wc = std::max<uint32_t>((maxn + 31) / 32, 1);
            CUDA_TRY(cudaMalloc(&d->d_bounds, (nranks + 1) * 4));
            CUDA_TRY(cudaMemcpy(d->d_bounds, d->bounds.data(), (nranks + 1) * 4, cudaMemcpyHostToDevice));
            if (uid != nullptr) {
                ncclUniqueId id;
                memcpy(&id, uid, sizeof(id));
                ncclComm_t c = nullptr;
                CUDA_TRY(cudaSetDevice(g->device));
                nccl_try(nccl().comm_init_rank(&c, nranks, id, rank), "ncclCommInitRank");
                d->comm = c;
            }
            g->joint_on = false;  // the joint node-major layout is a single-GPU batch mode
        }
    } catch (...) {
        if (d->d_bounds) cudaFree(d->d_bounds);
        delete d;
        throw;
    }
    g->dist = d;
}

uint32_t *dist_exchange_buffer(riki_graph *g, size_t chunk_words) {
    DistState *d = g->dist;
    const size_t need = chunk_words * d->nranks;
    if (need > d->x_words) {
        if (d->d_x) CUDA_TRY(cudaFree(d->d_x));
        d->d_x = nullptr;
        d->x_words = 0;
        size_t cap = std::max(need, d->x_words * 2);
        if (cudaMalloc(&d->d_x, cap * 4) != cudaSuccess) {
            cudaGetLastError();
            RIKI_THROW(RIKI_ENOMEM, "vertex-partitioned exchange buffer");
        }
        d->x_words = cap;
    }
    return d->d_x;
}

// In-place all-gather: rank r's slice is x + r*chunk_words.  Simulated partitions already
// wrote every slice into this buffer, and a 1-rank communicator is the identity as well.
void dist_allgather(riki_graph *g, uint32_t *x, size_t chunk_words, cudaStream_t s) {
    DistState *d = g->dist;
    d->exchanges++;
    d->exchanged_bytes += chunk_words * 4 * (size_t)d->nranks;
    if (!d->comm) return;
    nccl_try(nccl().all_gather(x + chunk_words * d->rank, x, chunk_words * 4, ncclUint8, (ncclComm_t)d->comm, s),
             "ncclAllGather");
}

// ---------------------------------------------------------------- vertex-partitioned push
// Real multi-rank runs: every rank owns three slices (levels rotate through them mod 3) in
// one allocation whose CUDA IPC handle is all-gathered once, so a rank's expansion kernel ORs
// bits straight into the owner's slice over NVLink (peer stores, no staging).  Level t:
//   push kernels (remote atomicOr into slice t mod 3)  ->  barrier (1-int all-reduce: every
//   rank's kernel has finished, so its remote writes are complete)  ->  all-gather of the
//   owned slices  ->  the owner clears slice (t + 2) mod 3 (written two levels on; any rank
//   reaching that level has passed this level's all-gather, which follows this clear).
// Simulated partitions and a single rank: one buffer [nranks][slice], cleared per level, and
// the exchange is the identity.
static void push_free(DistState *d) {
    for (size_t r = 0; r < d->peer_bases.size(); r++)
        if (d->peer_bases[r] && (int)r != d->rank) cudaIpcCloseMemHandle(d->peer_bases[r]);
    d->peer_bases.clear();
    if (d->d_slices) cudaFree(d->d_slices);
    if (d->d_gather) cudaFree(d->d_gather);
    if (d->d_xs) cudaFree(d->d_xs);
    if (d->d_one) cudaFree(d->d_one);
    d->d_slices = d->d_gather = nullptr;
    d->d_xs = nullptr;
    d->d_one = nullptr;
    d->slice_words = 0;
}

static bool push_real(const DistState *d) { return d->comm != nullptr && d->nranks > 1; }

void dist_push_setup(riki_graph *g, uint32_t slots) {
    DistState *d = g->dist;
    const size_t need = (size_t)std::max<uint32_t>(slots, 1) * 8 * d->wc;
    if (need <= d->slice_words) return;
    push_free(d);  // (collective in real mode: every rank grows at the same batch, same slots)
    const int P = d->nranks;
    auto alloc = [](void **p, size_t bytes, const char *what) {
        if (cudaMalloc(p, bytes) != cudaSuccess) {
            cudaGetLastError();
            RIKI_THROW(RIKI_ENOMEM, std::string("vertex-partitioned push: ") + what);
        }
    };
    std::vector<uint32_t *> xs(3 * (size_t)P);
    if (!push_real(d)) {
        alloc((void **)&d->d_slices, need * 4 * P, "slices");
        CUDA_TRY(cudaMemset(d->d_slices, 0, need * 4 * P));
        for (int k = 0; k < 3; k++)
            for (int r = 0; r < P; r++) xs[(size_t)k * P + r] = d->d_slices + need * r;
    } else {
        alloc((void **)&d->d_slices, need * 4 * 3, "own slices");
        CUDA_TRY(cudaMemset(d->d_slices, 0, need * 4 * 3));
        alloc((void **)&d->d_gather, need * 4 * P, "gather buffer");
        alloc((void **)&d->d_one, 4 * (size_t)P, "barrier");
        // all-gather the 64-byte IPC handles of every rank's slices, then map the peers'
        cudaIpcMemHandle_t h;
        CUDA_TRY(cudaIpcGetMemHandle(&h, d->d_slices));
        uint8_t *dh = nullptr;
        alloc((void **)&dh, sizeof(h) * P, "handle exchange");
        CUDA_TRY(cudaMemcpy(dh + sizeof(h) * d->rank, &h, sizeof(h), cudaMemcpyHostToDevice));
        nccl_try(nccl().all_gather(dh + sizeof(h) * d->rank, dh, sizeof(h), ncclUint8, (ncclComm_t)d->comm, 0),
                 "ncclAllGather (IPC handles)");
        std::vector<cudaIpcMemHandle_t> hs(P);
        CUDA_TRY(cudaMemcpy(hs.data(), dh, sizeof(h) * P, cudaMemcpyDeviceToHost));  // (syncs the NCCL call)
        cudaFree(dh);
        d->peer_bases.assign(P, nullptr);
        for (int r = 0; r < P; r++) {
            if (r == d->rank) { d->peer_bases[r] = d->d_slices; continue; }
            CUDA_TRY(cudaIpcOpenMemHandle(&d->peer_bases[r], hs[r], cudaIpcMemLazyEnablePeerAccess));
        }
        for (int k = 0; k < 3; k++)
            for (int r = 0; r < P; r++) xs[(size_t)k * P + r] = (uint32_t *)d->peer_bases[r] + need * k;
    }
    alloc((void **)&d->d_xs, xs.size() * sizeof(uint32_t *), "pointer table");
    CUDA_TRY(cudaMemcpy(d->d_xs, xs.data(), xs.size() * sizeof(uint32_t *), cudaMemcpyHostToDevice));
    d->slice_words = need;
    d->t = 0;
    d->used[0] = d->used[1] = d->used[2] = 0;
}

uint32_t *const *dist_push_targets(riki_graph *g) {
    DistState *d = g->dist;
    return d->d_xs + (push_real(d) ? (size_t)(d->t % 3) * d->nranks : 0);
}

const uint32_t *dist_push_exchange(riki_graph *g, size_t chunk, cudaStream_t s, size_t *stride) {
    DistState *d = g->dist;
    d->exchanges++;
    d->exchanged_bytes += chunk * 4 * (size_t)d->nranks;
    if (!push_real(d)) {
        *stride = d->slice_words;
        return d->d_slices;
    }
    const uint32_t k = (uint32_t)(d->t % 3);
    nccl_try(nccl().all_reduce(d->d_one, d->d_one, 1, ncclInt32, ncclSum, (ncclComm_t)d->comm, s), "ncclAllReduce (barrier)");
    nccl_try(nccl().all_gather(d->d_slices + d->slice_words * k, d->d_gather, chunk * 4, ncclUint8, (ncclComm_t)d->comm, s),
             "ncclAllGather (bit planes)");
    const uint32_t k2 = (uint32_t)((d->t + 2) % 3);
    if (d->used[k2]) CUDA_TRY(cudaMemsetAsync(d->d_slices + d->slice_words * k2, 0, d->used[k2] * 4, s));
    d->used[k2] = 0;
    d->used[k] = chunk;
    d->t++;
    *stride = chunk;
    return d->d_gather;
}

void dist_free(riki_graph *g) {
    DistState *d = g->dist;
    if (!d) return;
    push_free(d);
    if (d->comm) nccl().comm_destroy((ncclComm_t)d->comm);
    if (d->d_bounds) cudaFree(d->d_bounds);
    if (d->d_x) cudaFree(d->d_x);
    delete d;
    g->dist = nullptr;
}
