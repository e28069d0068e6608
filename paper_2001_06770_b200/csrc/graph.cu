// graph.cu -- graph residency and edge activation levels (a1/a2 of the hot-path table;
// not timed).  P:339-340 (CSR in GPU memory), P:189-217 (weighting and coarsening).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <string>

#include "internal.cuh"

namespace {

template <class T> T *dmalloc(size_t n, uint64_t *acc = nullptr) {
    T *p = nullptr;
    if (n == 0) n = 1;
    cudaError_t e = cudaMalloc(&p, n * sizeof(T));
    if (e != cudaSuccess) {
        cudaGetLastError();
        RIKI_THROW(RIKI_ENOMEM, "cudaMalloc of " + std::to_string(n * sizeof(T)) + " bytes failed");
    }
    if (acc) *acc += n * sizeof(T);
    return p;
}

int bits_for(uint64_t x) {
    int b = 1;
    while ((1ull << b) <= x) b++;
    return b;
}

__global__ void k_histogram(const uint32_t *key, uint64_t n, uint32_t *cnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(&cnt[key[i] + 1], 1u);
}

// Eq. 1-3, half-up rounding (R1), fp64 in the oracle's exact operation order
// with explicit round-to-nearest intrinsics so no FMA contraction can occur (R5).
__device__ __forceinline__ uint32_t coarsen_dev(double w, double alpha, double avg) {
    double x;
    if (w <= alpha) x = __dsub_rn(avg, __ddiv_rn(__dmul_rn(avg, __dsub_rn(alpha, w)), alpha));
    else x = __dadd_rn(avg, __ddiv_rn(__dmul_rn(avg, __dsub_rn(w, alpha)), __dsub_rn(1.0, alpha)));
    return (uint32_t)floor(__dadd_rn(x, 0.5));
}

__global__ void k_coarsen_edges(const double *w, uint64_t n, double alpha, double avg, uint8_t *a, uint32_t *bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        double x = w[i];
        if (!(x >= 0.0 && x <= 1.0)) { atomicOr(bad, 1u); a[i] = 0xFF; continue; }
        a[i] = (uint8_t)coarsen_dev(x, alpha, avg);
    }
}

__global__ void k_coarsen_nodes(const double *w, const uint32_t *dst, const uint32_t *iperm, uint64_t n,
                                double alpha, double avg, uint8_t *a, uint32_t *bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        double x = w[iperm[dst[i]]];  // w is indexed by the caller's node id
        if (!(x >= 0.0 && x <= 1.0)) { atomicOr(bad, 1u); a[i] = 0xFF; continue; }
        a[i] = (uint8_t)coarsen_dev(x, alpha, avg);
    }
}

// R29 (tie-break): the fine weight of every caller edge as the exact integer
// round(w * 2^32) (w * 2^32 is exact in fp64), so weight sums are order independent.
__global__ void k_wfix(const double *w, const uint32_t *dst, const uint32_t *iperm, uint64_t n,
                       unsigned long long *out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        double x = dst ? w[iperm[dst[i]]] : w[i];  // node variant: w of the edge's target
        out[i] = (unsigned long long)floor(__dadd_rn(__dmul_rn(x, 4294967296.0), 0.5));
    }
}

__global__ void k_make_keys(const uint32_t *node, const uint32_t *cls, uint64_t n, uint64_t *key, uint32_t *val) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        key[i] = (uint64_t)node[i] << 32 | cls[i];
        val[i] = (uint32_t)i;
    }
}

// run length of sorted key[i] by exponential + binary search around i
__global__ void k_run_length(const uint64_t *key, const uint32_t *eid, uint64_t n, uint32_t *cnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t k = key[i];
        // lower bound in [0, i]
        uint64_t step = 1, lo_out = i;  // key[lo_out] == k
        while (step <= lo_out && key[lo_out - step] == k) { lo_out -= step; step <<= 1; }
        uint64_t lo = step <= lo_out ? lo_out - step : 0, hi = lo_out;  // first equal in (lo, hi]
        while (lo < hi) { uint64_t m = (lo + hi) / 2; if (key[m] < k) lo = m + 1; else hi = m; }
        uint64_t first = lo;
        step = 1; uint64_t hi_in = i;
        while (hi_in + step < n && key[hi_in + step] == k) { hi_in += step; step <<= 1; }
        lo = hi_in; hi = (hi_in + step < n) ? hi_in + step : n;  // last equal in [lo, hi)
        while (lo + 1 < hi) { uint64_t m = (lo + hi) / 2; if (key[m] == k) lo = m; else hi = m; }
        cnt[eid[i]] = (uint32_t)(lo - first + 1);
    }
}

// P:193 raw weight = ln(count_out + count_in) of the integer count (R2: natural log), as the
// CORRECTLY ROUNDED fp64 value of ln n (R31), so that it has one definition independent of any
// math library: CUDA's log() is within 1 ulp and glibc's within ~0.52 ulp, and they disagree
// on ~1 in 10^5 integers (riki_debug_ln_table + tests/test_gpu_boundary.py).  Computed in
// double-double arithmetic (~2^-100 relative): n = 2^k * m, m in [sqrt(1/2), sqrt(2)),
// ln n = k ln 2 + 2 atanh(z), z = (m - 1)/(m + 1), |z| < 0.172, atanh by its series to z^49;
// the final hi + lo rounds to nearest.  Every operation is an explicit _rn intrinsic (no FMA
// contraction may touch the error-free transforms).
struct dd { double hi, lo; };
__device__ __forceinline__ dd dd_two_sum(double a, double b) {
    const double s = __dadd_rn(a, b), bb = __dsub_rn(s, a);
    return {s, __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb))};
}
__device__ __forceinline__ dd dd_fast(double a, double b) {  // |a| >= |b|
    const double s = __dadd_rn(a, b);
    return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd dd_add(dd a, dd b) {
    dd s = dd_two_sum(a.hi, b.hi), t = dd_two_sum(a.lo, b.lo);
    s.lo = __dadd_rn(s.lo, t.hi);
    s = dd_fast(s.hi, s.lo);
    s.lo = __dadd_rn(s.lo, t.lo);
    return dd_fast(s.hi, s.lo);
}
__device__ __forceinline__ dd dd_mul(dd a, dd b) {
    const double p = __dmul_rn(a.hi, b.hi);
    double e = __fma_rn(a.hi, b.hi, -p);
    e = __dadd_rn(e, __dadd_rn(__dmul_rn(a.hi, b.lo), __dmul_rn(a.lo, b.hi)));
    return dd_fast(p, e);
}
__device__ __forceinline__ dd dd_neg(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd dd_div(dd a, dd b) {  // three correction steps
    const double q1 = __ddiv_rn(a.hi, b.hi);
    dd r = dd_add(a, dd_neg(dd_mul({q1, 0.0}, b)));
    const double q2 = __ddiv_rn(r.hi, b.hi);
    r = dd_add(r, dd_neg(dd_mul({q2, 0.0}, b)));
    const double q3 = __ddiv_rn(r.hi, b.hi);
    return dd_add(dd_fast(q1, q2), {q3, 0.0});
}
__device__ __noinline__ double raw_ln(uint64_t n) {
    if (n <= 1) return 0.0;
    int k = 0;
    double m = frexp((double)n, &k);  // n < 2^53: exact; m in [0.5, 1)
    if (m < 0.70710678118654752440) { m = __dmul_rn(m, 2.0); k -= 1; }
    const dd z = dd_div({__dsub_rn(m, 1.0), 0.0}, {__dadd_rn(m, 1.0), 0.0});  // m -+ 1 exact
    const dd z2 = dd_mul(z, z);
    dd s = {0.0, 0.0};
    for (int i = 24; i >= 0; i--) s = dd_add(dd_mul(s, z2), dd_div({1.0, 0.0}, {(double)(2 * i + 1), 0.0}));
    const dd lnm = dd_mul(dd_mul(s, z), {2.0, 0.0});
    const dd LN2 = {6.93147180559945286227e-01, 2.31904681384629955842e-17};
    const dd r = dd_add(dd_mul({(double)k, 0.0}, LN2), lnm);
    return __dadd_rn(r.hi, r.lo);
}

__global__ void k_raw_weight(const uint32_t *co, const uint32_t *ci, uint64_t n, double *raw) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        raw[i] = raw_ln((uint64_t)co[i] + ci[i]);
}

__global__ void k_ln_table(uint64_t n0, uint64_t count, double *out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = raw_ln(n0 + i);
}

// P:194 min-max rescale; degenerate max == min -> 0 (R2)
__global__ void k_rescale(const double *raw, uint64_t n, const double *mnmx, double *w) {
    double mn = mnmx[0], mx = mnmx[1];
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        w[i] = (mx == mn) ? 0.0 : __ddiv_rn(__dsub_rn(raw[i], mn), __dsub_rn(mx, mn));
}

__global__ void k_act_keys(const uint32_t *node, const uint8_t *a, uint64_t n, uint64_t *key, uint32_t *val) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        key[i] = (uint64_t)node[i] << 8 | a[i];
        val[i] = (uint32_t)i;
    }
}

__global__ void k_gather_out(const uint64_t *key, const uint32_t *eid, const uint32_t *dst, uint64_t n,
                             uint32_t *col, uint8_t *act) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        col[i] = dst[eid[i]];
        act[i] = (uint8_t)(key[i] & 0xFF);
    }
}

__global__ void k_gather_in(const uint64_t *key, const uint32_t *eid, const uint32_t *src, uint64_t n,
                            uint32_t *isrc, uint32_t *ieid, uint8_t *iact) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t e = eid[i];
        isrc[i] = src[e];
        ieid[i] = e;
        iact[i] = (uint8_t)(key[i] & 0xFF);
    }
}

// Node descriptor: one 16-byte load gives the row start, the degree and, for rows of at most
// 8 edges, all their (sorted) activations packed in bytes (padding 0xFF), so the expansion
// finds the gate ranges a <= l / a == l with byte-SIMD compares instead of a binary search.
// Longer rows get a slot in the gate offset table (AOFF_LEVELS entries, see internal.cuh).
__device__ __forceinline__ uint32_t ub_act(const uint8_t *act, uint32_t lo, uint32_t hi, uint32_t k) {
    while (lo < hi) {  // first index with act > k
        uint32_t m = (lo + hi) >> 1;
        if (act[m] <= k) lo = m + 1; else hi = m;
    }
    return lo;
}
__global__ void k_desc(const uint32_t *row, const uint8_t *act, uint32_t V, uint4 *desc, uint32_t *aoff,
                       uint32_t *ncnt) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
        uint32_t rb = row[v], deg = row[v + 1] - rb;
        uint32_t lo = 0xFFFFFFFFu, hi = 0xFFFFFFFFu;
        if (deg <= 8) {
            for (uint32_t i = 0; i < deg; i++) {
                uint32_t b = act[rb + i];
                if (i < 4) lo = (lo & ~(0xFFu << (8 * i))) | (b << (8 * i));
                else hi = (hi & ~(0xFFu << (8 * (i - 4)))) | (b << (8 * (i - 4)));
            }
        } else {
            lo = atomicAdd(ncnt, 1u);  // table slot (any order: only the mapping matters)
            hi = 0;
            uint32_t *t = aoff + (size_t)lo * AOFF_LEVELS;
            uint32_t b = rb;
            for (uint32_t k = 0; k < AOFF_LEVELS; k++) t[k] = b = ub_act(act, b, rb + deg, k);
        }
        desc[v] = make_uint4(rb, deg, lo, hi);
    }
}
__global__ void k_count_long_rows(const uint32_t *row, uint32_t V, uint32_t *cnt) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x)
        if (row[v + 1] - row[v] > 8) atomicAdd(cnt, 1u);
}

// Node relabeling for L2 locality: internal id = rank by total degree (descending, then
// caller id).  In a power-law graph most edge endpoints are hubs, so the H words that the
// expansion hits most often form a short prefix of every query's H array.
__global__ void k_degree(const uint32_t *src, const uint32_t *dst, uint64_t n, uint32_t *deg) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        atomicAdd(&deg[src[i]], 1u);
        atomicAdd(&deg[dst[i]], 1u);
    }
}
__global__ void k_deg_keys(const uint32_t *deg, uint32_t V, uint64_t *key) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x)
        key[v] = (uint64_t)(0xFFFFFFFFu - deg[v]) << 32 | v;
}
__global__ void k_perm(const uint64_t *sorted, uint32_t V, uint32_t *perm, uint32_t *iperm) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < V; r += gridDim.x * blockDim.x) {
        uint32_t v = (uint32_t)sorted[r];
        perm[v] = r;
        iperm[r] = v;
    }
}
__global__ void k_count_heavy(const uint32_t *deg, uint32_t V, uint32_t thr, uint32_t *cnt) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x)
        if (deg[v] > thr) atomicAdd(cnt, 1u);
}
__global__ void k_relabel(uint32_t *x, uint64_t n, const uint32_t *perm) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        x[i] = perm[x[i]];
}

__global__ void k_minmax_pair(double *mnmx, const double *mn, const double *mx) {
    mnmx[0] = *mn;
    mnmx[1] = *mx;
}

unsigned grid_for(uint64_t n) { return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148ull * 16)); }

void sync_check(cudaStream_t s) { CUDA_TRY(cudaStreamSynchronize(s)); }

// Sort (key, eid) pairs by key over [0, end_bit); returns device buffers (caller frees).
void sort_pairs(cudaStream_t s, uint64_t *&keys, uint32_t *&vals, uint64_t n, int end_bit) {
    uint64_t *k2 = dmalloc<uint64_t>(n);
    uint32_t *v2 = dmalloc<uint32_t>(n);
    size_t tmp = 0;
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, k2, vals, v2, (int64_t)n, 0, end_bit, s));
    void *t = dmalloc<uint8_t>(tmp);
    CUDA_TRY(cub::DeviceRadixSort::SortPairs(t, tmp, keys, k2, vals, v2, (int64_t)n, 0, end_bit, s));
    sync_check(s);
    cudaFree(t);
    cudaFree(keys);
    cudaFree(vals);
    keys = k2;
    vals = v2;
}

// Builds both CSRs from d_act_e (activation by edge id): rows sorted by (activation, edge id).
void build_csr(riki_graph *g) {
    cudaStream_t s = g->stream;
    uint64_t E = g->E;
    int eb = bits_for(g->V) + 8;
    uint64_t *keys = dmalloc<uint64_t>(E);
    uint32_t *vals = dmalloc<uint32_t>(E);
    // out-CSR
    k_act_keys<<<grid_for(E), 256, 0, s>>>(g->d_src, g->d_act_e, E, keys, vals);
    sort_pairs(s, keys, vals, E, eb);
    k_gather_out<<<grid_for(E), 256, 0, s>>>(keys, vals, g->d_dst, E, g->d_col, g->d_act);
    {
        uint32_t *ncnt = dmalloc<uint32_t>(1);
        CUDA_TRY(cudaMemsetAsync(ncnt, 0, 4, s));
        k_desc<<<grid_for(g->V), 256, 0, s>>>(g->d_row, g->d_act, g->V, g->d_desc, g->d_aoff, ncnt);
        sync_check(s);
        cudaFree(ncnt);
    }
    // in-CSR
    k_act_keys<<<grid_for(E), 256, 0, s>>>(g->d_dst, g->d_act_e, E, keys, vals);
    sort_pairs(s, keys, vals, E, eb);
    k_gather_in<<<grid_for(E), 256, 0, s>>>(keys, vals, g->d_src, E, g->d_isrc, g->d_ieid, g->d_iact);
    {
        uint32_t *ncnt = dmalloc<uint32_t>(1);
        CUDA_TRY(cudaMemsetAsync(ncnt, 0, 4, s));
        k_desc<<<grid_for(g->V), 256, 0, s>>>(g->d_irow, g->d_iact, g->V, g->d_idesc, g->d_iaoff, ncnt);
        sync_check(s);
        cudaFree(ncnt);
    }
    sync_check(s);
    cudaFree(keys);
    cudaFree(vals);
    g->has_act = true;
}

void row_pointers(cudaStream_t s, const uint32_t *key, uint64_t E, uint32_t V, uint32_t *row) {
    CUDA_TRY(cudaMemsetAsync(row, 0, (V + 1) * sizeof(uint32_t), s));
    k_histogram<<<grid_for(E), 256, 0, s>>>(key, E, row);
    size_t tmp = 0;
    CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, tmp, row, row, (int)(V + 1), s));
    void *t = dmalloc<uint8_t>(tmp);
    CUDA_TRY(cub::DeviceScan::InclusiveSum(t, tmp, row, row, (int)(V + 1), s));
    sync_check(s);
    cudaFree(t);
}

void check_params(double alpha, double avg) {
    if (!(alpha > 0.0 && alpha < 1.0)) RIKI_THROW(RIKI_EINVAL, "alpha must be in (0,1) (P:198)");
    if (!(avg > 0.0) || !(2.0 * avg + 0.5 < 254.0)) RIKI_THROW(RIKI_EINVAL, "avg_hops must be in (0, 126.75)");
}

}  // namespace

// riki_load_graph_device: the caller's arrays are validated where they live.  bad: bit 0 =
// endpoint out of range, bit 1 = posting out of range, bit 2 = postings not sorted unique.
__global__ void k_validate_edges(const uint32_t *src, const uint32_t *dst, uint64_t E, uint32_t V, uint32_t *bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < E; i += (uint64_t)gridDim.x * blockDim.x)
        if (src[i] >= V || dst[i] >= V) atomicOr(bad, 1u);
}
__global__ void k_validate_postings(const uint64_t *tptr, uint32_t n_terms, const uint32_t *post, uint32_t V,
                                    uint32_t *bad) {
    for (uint32_t t = blockIdx.x; t < n_terms; t += gridDim.x)
        for (uint64_t i = tptr[t] + threadIdx.x; i < tptr[t + 1]; i += blockDim.x) {
            if (post[i] >= V) atomicOr(bad, 2u);
            if (i > tptr[t] && post[i] <= post[i - 1]) atomicOr(bad, 4u);
        }
}

void graph_load(riki_graph *g, uint32_t V, uint64_t E, const uint32_t *src, const uint32_t *dst, const uint32_t *cls,
                uint32_t n_terms, const uint64_t *tptr_in, const uint32_t *post, bool device_inputs) {
    if (V == 0) RIKI_THROW(RIKI_EINVAL, "n_nodes must be > 0");
    if (E >= (1ull << 32)) RIKI_THROW(RIKI_EINVAL, "n_edges must be < 2^32");
    if (E && (!src || !dst)) RIKI_THROW(RIKI_EINVAL, "null edge arrays");
    if (n_terms && (!tptr_in)) RIKI_THROW(RIKI_EINVAL, "null term_ptr");
    CUDA_TRY(cudaSetDevice(g->device));
    std::vector<uint64_t> tptr_h;
    const uint64_t *tptr = tptr_in;
    if (device_inputs && n_terms) {  // the (small) term pointer is needed on the host anyway (h_tptr)
        tptr_h.resize(n_terms + 1);
        CUDA_TRY(cudaMemcpy(tptr_h.data(), tptr_in, (n_terms + 1) * 8, cudaMemcpyDeviceToHost));
        tptr = tptr_h.data();
    }
    if (!device_inputs)
        for (uint64_t e = 0; e < E; e++)
            if (src[e] >= V || dst[e] >= V) RIKI_THROW(RIKI_EINVAL, "edge " + std::to_string(e) + " endpoint out of range");
    uint64_t P = n_terms ? tptr[n_terms] : 0;
    if (n_terms && tptr[0] != 0) RIKI_THROW(RIKI_EINVAL, "term_ptr[0] must be 0");
    if (P && !post) RIKI_THROW(RIKI_EINVAL, "null postings");
    for (uint32_t t = 0; t < n_terms; t++) {
        if (tptr[t + 1] < tptr[t]) RIKI_THROW(RIKI_EINVAL, "term_ptr not monotone");
        if (device_inputs) continue;
        for (uint64_t i = tptr[t]; i < tptr[t + 1]; i++) {
            if (post[i] >= V) RIKI_THROW(RIKI_EINVAL, "posting node out of range (term " + std::to_string(t) + ")");
            if (i > tptr[t] && post[i] <= post[i - 1])
                RIKI_THROW(RIKI_EINVAL, "postings of term " + std::to_string(t) + " not sorted unique");
        }
    }
    if (device_inputs) {
        uint32_t *bad = dmalloc<uint32_t>(1), hbad = 0;
        CUDA_TRY(cudaMemset(bad, 0, 4));
        if (E) k_validate_edges<<<grid_for(E), 256>>>(src, dst, E, V, bad);
        if (P) k_validate_postings<<<std::min<uint32_t>(n_terms, 148 * 16), 256>>>(tptr_in, n_terms, post, V, bad);
        CUDA_TRY(cudaMemcpy(&hbad, bad, 4, cudaMemcpyDeviceToHost));
        cudaFree(bad);
        if (hbad & 1) RIKI_THROW(RIKI_EINVAL, "edge endpoint out of range");
        if (hbad & 2) RIKI_THROW(RIKI_EINVAL, "posting node out of range");
        if (hbad & 4) RIKI_THROW(RIKI_EINVAL, "postings not sorted unique");
    }
    const cudaMemcpyKind kind = device_inputs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CUDA_TRY(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    g->V = V;
    g->E = E;
    g->n_terms = n_terms;
    uint64_t *acc = &g->graph_bytes;
    g->d_src = dmalloc<uint32_t>(E, acc);
    g->d_dst = dmalloc<uint32_t>(E, acc);
    g->d_cls = dmalloc<uint32_t>(E, acc);
    g->d_act_e = dmalloc<uint8_t>(E, acc);
    g->d_row = dmalloc<uint32_t>(V + 1, acc);
    g->d_col = dmalloc<uint32_t>(E, acc);
    g->d_act = dmalloc<uint8_t>(E, acc);
    g->d_desc = dmalloc<uint4>(V, acc);
    g->d_irow = dmalloc<uint32_t>(V + 1, acc);
    g->d_isrc = dmalloc<uint32_t>(E, acc);
    g->d_ieid = dmalloc<uint32_t>(E, acc);
    g->d_iact = dmalloc<uint8_t>(E, acc);
    g->d_tptr = dmalloc<uint64_t>(n_terms + 1, acc);
    g->d_post = dmalloc<uint32_t>(P, acc);
    cudaStream_t s = g->stream;
    if (E) {
        CUDA_TRY(cudaMemcpyAsync(g->d_src, src, E * 4, kind, s));
        CUDA_TRY(cudaMemcpyAsync(g->d_dst, dst, E * 4, kind, s));
        if (cls) CUDA_TRY(cudaMemcpyAsync(g->d_cls, cls, E * 4, kind, s));
        else CUDA_TRY(cudaMemsetAsync(g->d_cls, 0, E * 4, s));
    }
    g->h_tptr.assign(n_terms + 1, 0);
    if (n_terms) {
        std::copy(tptr, tptr + n_terms + 1, g->h_tptr.begin());
        CUDA_TRY(cudaMemcpyAsync(g->d_tptr, tptr, (n_terms + 1) * 8, cudaMemcpyHostToDevice, s));
        if (P) CUDA_TRY(cudaMemcpyAsync(g->d_post, post, P * 4, kind, s));
    }
    // ---- degree-descending relabeling (internal ids); translated back at the boundary
    g->d_perm = dmalloc<uint32_t>(V, acc);
    g->d_iperm = dmalloc<uint32_t>(V, acc);
    {
        uint32_t *deg = dmalloc<uint32_t>(V);
        uint64_t *k1 = dmalloc<uint64_t>(V), *k2 = dmalloc<uint64_t>(V);
        CUDA_TRY(cudaMemsetAsync(deg, 0, (size_t)V * 4, s));
        if (E) k_degree<<<grid_for(E), 256, 0, s>>>(g->d_src, g->d_dst, E, deg);
        k_deg_keys<<<grid_for(V), 256, 0, s>>>(deg, V, k1);
        size_t tmp = 0;
        CUDA_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tmp, k1, k2, (int64_t)V, 0, 64, s));
        void *t = dmalloc<uint8_t>(tmp);
        CUDA_TRY(cub::DeviceRadixSort::SortKeys(t, tmp, k1, k2, (int64_t)V, 0, 64, s));
        k_perm<<<grid_for(V), 256, 0, s>>>(k2, V, g->d_perm, g->d_iperm);
        uint32_t *cnt = dmalloc<uint32_t>(1);
        CUDA_TRY(cudaMemsetAsync(cnt, 0, 4, s));
        // total degree = 2 x in-degree in the bidirected graph; heavy = in-degree > 32
        k_count_heavy<<<grid_for(V), 256, 0, s>>>(deg, V, 64, cnt);
        CUDA_TRY(cudaMemcpyAsync(&g->Vh, cnt, 4, cudaMemcpyDeviceToHost, s));
        sync_check(s);
        cudaFree(cnt);
        if (E) {
            k_relabel<<<grid_for(E), 256, 0, s>>>(g->d_src, E, g->d_perm);
            k_relabel<<<grid_for(E), 256, 0, s>>>(g->d_dst, E, g->d_perm);
        }
        if (P) k_relabel<<<grid_for(P), 256, 0, s>>>(g->d_post, P, g->d_perm);
        sync_check(s);
        cudaFree(t); cudaFree(deg); cudaFree(k1); cudaFree(k2);
    }
    row_pointers(s, g->d_src, E, V, g->d_row);
    row_pointers(s, g->d_dst, E, V, g->d_irow);
    {   // gate offset table for out-rows longer than 8 edges
        uint32_t *cnt = dmalloc<uint32_t>(1);
        CUDA_TRY(cudaMemsetAsync(cnt, 0, 4, s));
        k_count_long_rows<<<grid_for(V), 256, 0, s>>>(g->d_row, V, cnt);
        CUDA_TRY(cudaMemcpyAsync(&g->n_aoff, cnt, 4, cudaMemcpyDeviceToHost, s));
        sync_check(s);
        g->d_aoff = dmalloc<uint32_t>((size_t)std::max<uint32_t>(g->n_aoff, 1) * AOFF_LEVELS, acc);
        CUDA_TRY(cudaMemsetAsync(cnt, 0, 4, s));
        k_count_long_rows<<<grid_for(V), 256, 0, s>>>(g->d_irow, V, cnt);
        CUDA_TRY(cudaMemcpyAsync(&g->n_iaoff, cnt, 4, cudaMemcpyDeviceToHost, s));
        sync_check(s);
        g->d_iaoff = dmalloc<uint32_t>((size_t)std::max<uint32_t>(g->n_iaoff, 1) * AOFF_LEVELS, acc);
        g->d_idesc = dmalloc<uint4>(V, acc);
        cudaFree(cnt);
    }
    sync_check(s);
}

void graph_free(riki_graph *g) {
    void *ps[] = {g->d_src, g->d_dst, g->d_cls, g->d_act_e, g->d_row, g->d_col, g->d_act, g->d_desc,
                  g->d_irow, g->d_isrc, g->d_ieid, g->d_iact, g->d_tptr, g->d_post, g->d_perm, g->d_iperm, g->d_aoff, g->d_idesc, g->d_iaoff, g->d_wfix};
    for (void *p : ps) if (p) cudaFree(p);
    if (g->stream) cudaStreamDestroy(g->stream);
}

static void finish_act(riki_graph *g, uint32_t *d_bad) {
    uint32_t bad = 0;
    CUDA_TRY(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, g->stream));
    sync_check(g->stream);
    cudaFree(d_bad);
    if (bad) RIKI_THROW(RIKI_EINVAL, "weights must lie in [0,1] (P:194)");
    build_csr(g);
}

// Keeps the fine weights (fixed point, by caller edge id) for the tie-break (R29).
static void keep_wfix(riki_graph *g, const double *dw, const uint32_t *dst) {
    if (!g->d_wfix && g->E) g->d_wfix = dmalloc<unsigned long long>(g->E);
    if (g->E) k_wfix<<<grid_for(g->E), 256, 0, g->stream>>>(dw, dst, g->d_iperm, g->E, g->d_wfix);
}

void graph_set_edge_weights(riki_graph *g, const double *w01, double alpha, double avg) {
    check_params(alpha, avg);
    if (g->E && !w01) RIKI_THROW(RIKI_EINVAL, "null weights");
    double *dw = dmalloc<double>(g->E);
    uint32_t *bad = dmalloc<uint32_t>(1);
    CUDA_TRY(cudaMemsetAsync(bad, 0, 4, g->stream));
    if (g->E) CUDA_TRY(cudaMemcpyAsync(dw, w01, g->E * 8, cudaMemcpyHostToDevice, g->stream));
    k_coarsen_edges<<<grid_for(g->E), 256, 0, g->stream>>>(dw, g->E, alpha, avg, g->d_act_e, bad);
    keep_wfix(g, dw, nullptr);
    sync_check(g->stream);
    cudaFree(dw);
    finish_act(g, bad);
}

void graph_set_node_weights(riki_graph *g, const double *w01, double alpha, double avg) {
    check_params(alpha, avg);
    if (!w01) RIKI_THROW(RIKI_EINVAL, "null weights");
    double *dw = dmalloc<double>(g->V);
    uint32_t *bad = dmalloc<uint32_t>(1);
    CUDA_TRY(cudaMemsetAsync(bad, 0, 4, g->stream));
    CUDA_TRY(cudaMemcpyAsync(dw, w01, (size_t)g->V * 8, cudaMemcpyHostToDevice, g->stream));
    k_coarsen_nodes<<<grid_for(g->E), 256, 0, g->stream>>>(dw, g->d_dst, g->d_iperm, g->E, alpha, avg, g->d_act_e, bad);
    keep_wfix(g, dw, g->d_dst);
    sync_check(g->stream);
    cudaFree(dw);
    finish_act(g, bad);
}

void graph_set_label_weights(riki_graph *g, double alpha, double avg) {
    check_params(alpha, avg);
    cudaStream_t s = g->stream;
    uint64_t E = g->E;
    int eb = 32 + bits_for(g->V);
    uint32_t *co = dmalloc<uint32_t>(E), *ci = dmalloc<uint32_t>(E);
    uint64_t *keys = dmalloc<uint64_t>(E);
    uint32_t *vals = dmalloc<uint32_t>(E);
    // |{e_ix : same class}| over out-edges of v_i
    k_make_keys<<<grid_for(E), 256, 0, s>>>(g->d_src, g->d_cls, E, keys, vals);
    sort_pairs(s, keys, vals, E, eb);
    k_run_length<<<grid_for(E), 256, 0, s>>>(keys, vals, E, co);
    // |{e_xj : same class}| over in-edges of v_j
    k_make_keys<<<grid_for(E), 256, 0, s>>>(g->d_dst, g->d_cls, E, keys, vals);
    sort_pairs(s, keys, vals, E, eb);
    k_run_length<<<grid_for(E), 256, 0, s>>>(keys, vals, E, ci);
    sync_check(s);
    cudaFree(keys);
    cudaFree(vals);
    double *raw = dmalloc<double>(E), *w = dmalloc<double>(E), *mm = dmalloc<double>(4);
    k_raw_weight<<<grid_for(E), 256, 0, s>>>(co, ci, E, raw);
    size_t tmp = 0;
    CUDA_TRY(cub::DeviceReduce::Min(nullptr, tmp, raw, mm + 2, (int64_t)E, s));
    size_t tmp2 = 0;
    CUDA_TRY(cub::DeviceReduce::Max(nullptr, tmp2, raw, mm + 3, (int64_t)E, s));
    tmp = std::max(tmp, tmp2);
    void *t = dmalloc<uint8_t>(tmp);
    CUDA_TRY(cub::DeviceReduce::Min(t, tmp, raw, mm + 2, (int64_t)E, s));
    CUDA_TRY(cub::DeviceReduce::Max(t, tmp, raw, mm + 3, (int64_t)E, s));
    k_minmax_pair<<<1, 1, 0, s>>>(mm, mm + 2, mm + 3);
    k_rescale<<<grid_for(E), 256, 0, s>>>(raw, E, mm, w);
    uint32_t *bad = dmalloc<uint32_t>(1);
    CUDA_TRY(cudaMemsetAsync(bad, 0, 4, s));
    k_coarsen_edges<<<grid_for(E), 256, 0, s>>>(w, E, alpha, avg, g->d_act_e, bad);
    keep_wfix(g, w, nullptr);
    sync_check(s);
    cudaFree(t); cudaFree(raw); cudaFree(w); cudaFree(mm); cudaFree(co); cudaFree(ci);
    finish_act(g, bad);
}

void graph_set_act(riki_graph *g, const uint8_t *a) {
    if (g->E && !a) RIKI_THROW(RIKI_EINVAL, "null activation array");
    for (uint64_t e = 0; e < g->E; e++)
        if (a[e] == 0xFF) RIKI_THROW(RIKI_EINVAL, "activation 255 is reserved");
    if (g->E) CUDA_TRY(cudaMemcpyAsync(g->d_act_e, a, g->E, cudaMemcpyHostToDevice, g->stream));
    sync_check(g->stream);
    if (g->d_wfix) {  // activation levels without fine weights: no weight-sum tie-break (R29)
        cudaFree(g->d_wfix);
        g->d_wfix = nullptr;
    }
    build_csr(g);
}

void graph_get_act(const riki_graph *g, uint8_t *a) {
    if (!g->has_act) RIKI_THROW(RIKI_ENOWEIGHTS, "activation levels not set");
    if (g->E) CUDA_TRY(cudaMemcpyAsync(a, g->d_act_e, g->E, cudaMemcpyDeviceToHost, g->stream));
    sync_check(g->stream);
}

void graph_debug_ln_table(int device, uint64_t n0, uint64_t count, double *out_host) {
    CUDA_TRY(cudaSetDevice(device));
    double *d = nullptr;
    if (count == 0) return;
    CUDA_TRY(cudaMalloc(&d, count * sizeof(double)));
    k_ln_table<<<grid_for(count), 256>>>(n0, count, d);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpy(out_host, d, count * sizeof(double), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (e != cudaSuccess) RIKI_THROW(RIKI_ECUDA, std::string("ln table: ") + cudaGetErrorString(e));
}
