// engine.cu -- RIKI query engine on sm_100a: batched, level-synchronous two-run search.
//
//   run 1 (central keywords) and run 2 (marginal keywords), each:
//     seed -> per level: [attach + decide (run 2)] -> plan/terminate
//      -> Alg. 1 expansion with CF blocking
//   between the runs: candidate CGs (R13) sorted by (S^c, v) and recovered (Alg. 2,
//   P:503-561) by one CTA each; during run 2 every newly attached candidate is recovered
//   as an RPG and PTC-checked (Def. RPG, R19); finally the top-k by
//   (S^r, S^c, v) (Eq. 6, R23) are sorted and packed for the host.
//
// All queries of a batch advance in lock-step (one level per iteration), so every launch
// covers the frontiers of all in-flight queries.  H rows are one 32- or 64-bit word per
// node (byte = hitting level, 0xFF = inf); a relaxation is one atomicAnd that both writes
// l+1 into every still-infinite selected byte and tells the caller whether it was the
// first writer of the row at this level (enqueue) and whether it completed the row
// (identification at level l+1, R10).  Lock-free by Theorem lockfree.
#include <cuda_runtime.h>

#include <cub/device/device_segmented_radix_sort.cuh>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <chrono>
#include <functional>
#include <string>
#include <type_traits>
#include <vector>

#include "internal.cuh"

typedef unsigned __int128 u128;

namespace {

constexpr uint32_t MAX_SLOTS = 1024;
// H layout of the per-slot ("slot-major") mode: slots are grouped by HGRP, and inside a group
// the rows of one node are contiguous, so row (s, n) lives at
//   H + ((s / HGRP) * V + n) * HGRP + s % HGRP        (in rows);
// HGRP = 1 is plain slot-major.  Queries of a group that touch the same (hub) node share its
// sector.
#ifndef HGRP
#define HGRP 1
#endif
#ifndef LEVEL_BATCH
#define LEVEL_BATCH 4  // levels enqueued between host termination checks
#endif
#ifndef EXP_HEAVY
#define EXP_HEAVY 128
#endif
constexpr uint32_t HEAVY = EXP_HEAVY;  // longer active ranges are split into CHUNK-edge work items
constexpr uint32_t CHUNK = EXP_HEAVY;
constexpr uint32_t EMPTY = 0xFFFFFFFFu;
constexpr uint32_t SORT_SMEM = 8192;  // u32 keys sorted in shared memory
constexpr uint32_t U128_SORT_KEYS = 4096;  // u128 result keys sorted in shared memory (64 KB; larger sets in global)

enum Ctr { C_NHEAVY = 0, C_NNEWATT, C_NOVF, C_ACTIVE, C_TOTAL, C_NCAND_TOTAL, C_NOVF2, C_NPULL, C_JQN0, C_JQN1,
           C_JQCUR, C_JHEAVY, C_LEVEL, C_RECQ, C_NCTR = 16 };
// level argument of the per-level kernels: a value, or LV_DEVICE = read the device level
// counter ctr[C_LEVEL] (the whole-run CUDA graph with a device-side while loop)
constexpr uint32_t LV_DEVICE = 0xFFFFFFFFu;
enum Prof { P_ITEMS = 0, P_EDGES, P_NEWCELLS, P_ENQ, P_RELAX, P_PULLNODES, P_PULLEDGES, P_ITEMS_WORK,
            // recovery diagnostics (compiled in with -DREC_STATS=1)
            P_R_BUILDS = 8, P_R_BEDGES, P_R_BCYC, P_R_WAITS, P_R_WCYC, P_R_CANDS, P_R_CANDCYC, P_R_CANDMAX, P_R_BMAX,
            P_R_ITEMS, P_R_WARPMAX, P_R_H0,  // P_R_H0..+5: candidate-time histogram
            // expansion item diagnostics (compiled in with -DEXP_STATS=1)
            P_X_DUP = 24, P_X_BLOCKED, P_X_IDLE, P_X_WORK,
            P_ATOMS = 28,  // relaxation atomics issued by the expansion (random-access roofline)
            // recovery tier diagnostics (REC_STATS): candidates per tier, big-tier sizes
            P_R_T1 = 32, P_R_T2, P_R_T2NODES, P_R_T2EDGES, P_R_T2MAXE, P_R_T1RPG, P_R_T2RPG, P_NPROF = 40 };
#ifndef EXP_STATS
#define EXP_STATS 0
#endif
// cache policy of the expansion's streamed reads (CSR columns, queue entries): 0 = __ldg
// (default), 1 = __ldcs (evict-first: keep L2 for the random H-row accesses)
#ifndef EXP_STREAM_LD
#define EXP_STREAM_LD 0
#endif
#if EXP_STREAM_LD
#define STREAM_LD(p) __ldcs(p)
#else
#define STREAM_LD(p) __ldg(p)
#endif
#ifndef REC_STATS
#define REC_STATS 0
#endif
enum Err { E_CAND = 1, E_HEAVY = 2, E_ARENA = 4, E_EXTRACT = 8, E_OUT = 16, E_UNRESOLVED = 32, E_QUEUE = 64 };

struct SlotState {
    uint32_t T[2];
    uint32_t term[2][RIKI_MAX_TERMS];
    uint32_t k, w, depth;
    uint32_t beam_mode, ptc_mode, early_term, tie_break;
    double gamma;
    uint32_t in_phase, level;
    uint32_t nq[2];
    uint32_t blocking, collect, stop_m, pull, reached;  // reached: new-node events this run
    uint32_t ncand, ncand_kept, n_extract;
    int32_t L_end[2];
    unsigned long long relax[2];
    uint32_t n_attached, n_ptc_fail, nR, nres;
    uint32_t first_unatt, nR_sorted;  // run-2 bookkeeping (monotone cursor, sorted prefix of R)
    uint32_t err, active;
    uint32_t ntie;  // tie-break (R29): results [0, ntie) whose order needs the weight sums
};

struct Cand {
    uint32_t v, sc;
    uint32_t nodes_off, n_nodes, edges_off, n_edges, vc_off, n_vc;
    uint32_t attached, ptc, sm, ext;  // ext = caller id of v (ordering and output use caller ids)
    double sr;
    unsigned long long wsum;  // tie-break (R29): W(G^r) (W(CG) when M is empty)
    uint8_t mdist[RIKI_MAX_TERMS];
};

struct OutHdr {
    uint32_t central, sc, sm, ptc;
    double score;
    uint32_t n_nodes, nodes_off, n_edges, edges_off, n_vc, vc_off;
    uint8_t cdist[RIKI_MAX_TERMS], mdist[RIKI_MAX_TERMS];
};

// View of one query's H array: slot-major (row of node n at base + n) or node-major (all
// slots' rows of node n contiguous, stride SP rows) for the joint multi-query traversal.
template <class RowT> struct HV {
    RowT *base;
    uint32_t sn;
    __device__ __forceinline__ RowT *operator+(uint32_t n) const { return base + (size_t)n * sn; }
};

// Device view of the workspace (passed by value to every kernel).
struct WsDev {
    SlotState *st;
    uint32_t nslots, V, W, capc, kmax;
    uint8_t *H[2];
    uint32_t rb[2];
    uint32_t *q, *bm;
    uint32_t qcap;  // entries per level queue: V, or 2V after an overflow (a node can be retained and new)
    uint32_t *jq, *jbm;  // joint traversal: union frontier queues [2][V] and bit-packed flags [2][W]
    uint64_t *ck;
    Cand *cd;
    u128 *rk;
    unsigned long long *offs;  // frontier-item prefix over the slots (k_expand<.., WIDE> beyond 2^32)
    uint32_t *coffs, *pslots, *ppos;  // pull / VP slots: position -> slot, slot -> position
    uint32_t track_reached;  // direction-optimising mode: count new nodes per slot
    uint4 *heavy;
    uint32_t heavy_cap;
    uint32_t *ctr;
    unsigned long long *prof;
    uint32_t *arena;
    unsigned long long *arena_used, arena_cap;
    uint2 *newatt, *ovf, *ovf2;
    uint32_t ovf_cap;
    uint8_t *cst;  // per (slot, candidate): 0 unattached, 1 attached and pending RPG recovery,
                   // 2 recovered, 3 excluded from the top-k (never recovered); bounded mode
    uint32_t bounded;  // run 2 recovers RPGs in waves, only for candidates that can enter the top-k
    uint32_t *big;
    unsigned long long big_words;
    uint4 *mtab;
    OutHdr *hdr;
    uint2 *tie;  // tie-break scratch per slot (capc): (candidate, tie-group start)
    uint32_t *resid;
    uint32_t *out;
    unsigned long long *out_used, out_cap;

    __device__ __forceinline__ uint32_t *Q(uint32_t s, uint32_t b) const { return q + ((size_t)s * 2 + b) * qcap; }
    __device__ __forceinline__ uint32_t *JQ(uint32_t b) const { return jq + (size_t)b * V; }
    __device__ __forceinline__ uint32_t *JBM(uint32_t b) const { return jbm + (size_t)b * W; }
    uint32_t hnode, SP;  // H layout: 0 slot-major, 1 node-major with SP (padded) slots per node
    template <class RowT> __device__ __forceinline__ HV<RowT> Hs(int ph, uint32_t s) const {
        return hnode ? HV<RowT>{(RowT *)(H[ph] + (size_t)s * rb[ph]), SP}
                     : HV<RowT>{(RowT *)(H[ph] + ((size_t)(s / HGRP) * V * HGRP + s % HGRP) * rb[ph]), (uint32_t)HGRP};
    }
    __device__ __forceinline__ uint64_t *CK(uint32_t s) const { return ck + (size_t)s * capc; }
    __device__ __forceinline__ Cand *CD(uint32_t s) const { return cd + (size_t)s * capc; }
    __device__ __forceinline__ u128 *RK(uint32_t s) const { return rk + (size_t)s * capc; }
    __device__ __forceinline__ uint8_t *CST(uint32_t s) const { return cst + (size_t)s * capc; }
};

template <class RowT> __device__ __forceinline__ RowT used_mask(uint32_t T) {
    return T >= sizeof(RowT) ? (RowT)~(RowT)0 : (((RowT)1 << (8 * T)) - 1);
}
template <class RowT> __device__ __forceinline__ RowT vmin(RowT a, RowT b);
template <> __device__ __forceinline__ uint32_t vmin<uint32_t>(uint32_t a, uint32_t b) { return __vminu4(a, b); }
template <> __device__ __forceinline__ uint16_t vmin<uint16_t>(uint16_t a, uint16_t b) { return (uint16_t)__vminu4(a, b); }
template <> __device__ __forceinline__ uint64_t vmin<uint64_t>(uint64_t a, uint64_t b) {
    return (uint64_t)__vminu4((uint32_t)(a >> 32), (uint32_t)(b >> 32)) << 32 |
           __vminu4((uint32_t)a, (uint32_t)b);
}
template <class RowT> __device__ __forceinline__ RowT shfl(RowT v, int src) { return __shfl_sync(FULLMASK, v, src); }

// Eq. 6 in the oracle's exact operation order (R5): gamma*sc + (1-gamma)*sm.
__device__ __forceinline__ double rpg_score(double g, uint32_t sc, uint32_t sm) {
    return __dadd_rn(__dmul_rn(g, (double)sc), __dmul_rn(__dsub_rn(1.0, g), (double)sm));
}
__device__ __forceinline__ u128 rkey(double sr, uint32_t sc, uint32_t v) {
    return (u128)(unsigned long long)__double_as_longlong(sr) << 64 | (u128)sc << 32 | v;
}

template <class T> __device__ __forceinline__ uint32_t find_slot(const T *offs, uint32_t n, T item) {
    // largest s with offs[s] <= item (offs non-decreasing, offs[n] = total)
    uint32_t lo = 0, hi = n;
    while (hi - lo > 1) {
        uint32_t m = (lo + hi) >> 1;
        if (offs[m] <= item) lo = m; else hi = m;
    }
    return lo;
}

// Warp-uniform form: largest s < n with offs[s] <= item for the same `item` in every lane
// (n <= 32 * 32): a 32-way ballot over every stride-th boundary, then one over the stride.
template <class T> __device__ __forceinline__ uint32_t find_slot_warp(const T *offs, uint32_t n, T item) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t stride = (n + 31) >> 5;
    const uint32_t j = lane * stride;
    const uint32_t c = __popc(__ballot_sync(FULLMASK, j < n && offs[j] <= item)) - 1;
    const uint32_t j2 = c * stride + lane;
    return c * stride + __popc(__ballot_sync(FULLMASK, lane < stride && j2 < n && offs[j2] <= item)) - 1;
}

// ====================================================================== run setup
__global__ void k_phase_begin(WsDev w, int ph, int hitting_mode) {
    uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= w.nslots) return;
    SlotState &st = w.st[s];
    uint32_t T = st.T[ph];
    st.in_phase = st.active && T > 0 && !st.err;
    st.level = 0;
    st.nq[0] = st.nq[1] = 0;
    st.stop_m = 0;
    st.reached = 0;
    st.pull = 0;
    st.L_end[ph] = -1;
    if (hitting_mode >= 0) {  // debug boundary: 0 none, 1 central CF, 2 marginal stop rule
        st.blocking = hitting_mode == 1 || (hitting_mode == 2 && T >= 2);
        st.collect = 0;
    } else if (ph == 0) {
        st.blocking = 1;  // CF: "stop expanding a node once it is identified"
        st.collect = 1;
        st.ncand = 0;
    } else {
        st.blocking = T >= 2;  // stop rule P:373, disabled for |M| = 1 (R11)
        st.collect = 0;
        st.nR = 0;
        st.n_attached = 0;
        st.n_ptc_fail = 0;
        st.first_unatt = 0;
        st.nR_sorted = 0;
    }
}

// H rows: used bytes = 0xFF (inf), padding bytes = 0 (P:344 static initialisation)
template <class RowT> __global__ void k_fill_H(WsDev w, int ph) {
    uint32_t s = blockIdx.y;
    if (!w.st[s].in_phase) return;
    RowT pat = used_mask<RowT>(w.st[s].T[ph]);
    const HV<RowT> H = w.Hs<RowT>(ph, s);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < w.V; i += gridDim.x * blockDim.x) *(H + i) = pat;
}

// Node-major H (joint traversal): one 16-byte chunk per thread, slot patterns from shared
// memory; slots not in this run (or padding) get 0 (= complete and blocked: never touched).
template <class RowT> __global__ void k_fill_H_nodemajor(WsDev w, int ph) {
    __shared__ RowT pat[1024];
    for (uint32_t s = threadIdx.x; s < w.SP; s += blockDim.x) {
        RowT p = 0;
        if (s < w.nslots && w.st[s].in_phase) p = used_mask<RowT>(w.st[s].T[ph]);
        pat[s] = p;
    }
    __syncthreads();
    const uint32_t per = 16 / sizeof(RowT), chunks = w.SP / per;
    const uint64_t total = (uint64_t)w.V * chunks;
    uint4 *H = (uint4 *)w.H[ph];
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t c = (uint32_t)(i % chunks);
        RowT v[16 / sizeof(RowT)];
#pragma unroll
        for (uint32_t k = 0; k < per; k++) v[k] = pat[c * per + k];
        H[i] = *(uint4 *)v;
    }
}

// Seeds: h = 0 at keyword nodes, all keyword nodes are frontiers; level-0
// identification of nodes holding every phase keyword (score 0).
template <class RowT> __global__ void k_seed(GraphDev g, WsDev w, int ph) {
    uint32_t s = blockIdx.y;
    SlotState &st = w.st[s];
    if (!st.in_phase) return;
    const HV<RowT> H = w.Hs<RowT>(ph, s);
    const uint32_t T = st.T[ph];
    const RowT used = used_mask<RowT>(T);
    for (uint32_t j = 0; j < T; j++) {
        uint32_t t = st.term[ph][j];
        uint64_t b = g.tptr[t], e = g.tptr[t + 1];
        for (uint64_t i = b + blockIdx.x * blockDim.x + threadIdx.x; i < e; i += (uint64_t)gridDim.x * blockDim.x) {
            uint32_t v = g.post[i];
            RowT andm = ~((RowT)0xFF << (8 * j));
            RowT old = Row<RowT>::atomic_and(H + v, andm);
            RowT nw = old & andm;
            if ((Row<RowT>::eq(old, Row<RowT>::splat(0xFF)) & used) == used) {  // first seed of this node
                uint32_t p = atomicAdd(&st.nq[0], 1u);
                if (w.hnode) {  // joint traversal: union frontier, deduplicated by the bit-packed flags
                    uint32_t bit = 1u << (v & 31);
                    if (!(atomicOr(w.JBM(0) + (v >> 5), bit) & bit)) w.JQ(0)[atomicAdd(&w.ctr[C_JQN0], 1u)] = v;
                } else {
                    w.Q(s, 0)[p] = v;
                }
                atomicAdd(&st.reached, 1u);
            }
            if (st.collect && Row<RowT>::eq(nw, Row<RowT>::splat(0xFF)) == 0 &&
                Row<RowT>::byte(old, j) == 0xFF) {
                uint32_t p = atomicAdd(&st.ncand, 1u);
                if (p < w.capc) w.CK(s)[p] = (uint64_t)g.iperm[v];  // score 0
                else atomicOr(&st.err, (uint32_t)E_CAND);
            }
        }
    }
}

// ====================================================================== plan / terminate
// One block: per-slot termination check for level l, then an exclusive scan of the
// frontier sizes of the slots that expand (flattened work index for k_expand).
#ifndef PULL_ALPHA
#define PULL_ALPHA 14
#endif
#ifndef PULL_MIN_DIV
#define PULL_MIN_DIV 64
#endif
// pull_min: minimum frontier for bottom-up (0xFFFFFFFF disables it)
__global__ void k_plan(WsDev w, int ph, uint32_t l_arg, uint32_t pull_min) {
    const uint32_t l = l_arg == LV_DEVICE ? w.ctr[C_LEVEL] : l_arg;
    __shared__ unsigned long long sc[64];  // warp sums, then their inclusive prefix
    __shared__ uint32_t nact, wpull[MAX_SLOTS / 32];
    __shared__ unsigned long long nenq;
    uint32_t s = threadIdx.x;
    if (s == 0) { nact = 0; nenq = 0; }
    __syncthreads();
    uint32_t items = 0;
    bool pl = false;
    if (s < w.nslots) {
        SlotState &st = w.st[s];
        if (st.in_phase) {
            st.level = l;
            uint32_t cur = l & 1;
            // queue entries written by level l-1's expansion (profiling counter P_ENQ)
            if (l > 0 && !w.hnode && st.nq[cur]) atomicAdd(&nenq, (unsigned long long)st.nq[cur]);
            bool stop;
            if (ph == 0)  // P:362 ">= w CGs", depth bound (R8), empty frontier
                stop = st.ncand >= st.w || l >= st.depth || st.nq[cur] == 0;
            else
                stop = st.stop_m;
            if (stop || st.err) {
                st.in_phase = 0;
                st.L_end[ph] = (int32_t)l;
                st.pull = 0;
            } else {
                items = st.nq[cur];
                st.nq[cur ^ 1] = 0;
                atomicAdd(&nact, 1u);
                // direction-optimising (Beamer): bottom-up once the frontier is large compared
                // with what is still unvisited (estimate: V*T minus new-node events)
                uint64_t total = (uint64_t)w.V * st.T[ph];
                uint64_t unvisited = total > st.reached ? total - st.reached : 0;
                st.pull = pull_min == 0 || (items >= pull_min && (uint64_t)items * PULL_ALPHA > unvisited);
                pl = st.pull;
            }
        }
    }
    // pull slots in ascending slot order (a deterministic compaction, so every rank of the
    // vertex-partitioned mode maps exchange position p to the same slot)
    const uint32_t pb = __ballot_sync(FULLMASK, pl);
    if ((s & 31) == 0) wpull[s >> 5] = __popc(pb);
    __syncthreads();
    uint32_t pbefore = 0, npull = 0;
    for (uint32_t i = 0; i < MAX_SLOTS / 32; i++) {
        pbefore += i < (s >> 5) ? wpull[i] : 0;
        npull += wpull[i];
    }
    if (pl) w.pslots[pbefore + __popc(pb & lanemask_lt())] = s;
    if (s < w.nslots) w.ppos[s] = pl ? pbefore + __popc(pb & lanemask_lt()) : EMPTY;
    // block exclusive scan over MAX_SLOTS: warp shuffles, then one pass over the 32 warp sums
    unsigned long long incl = items;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(FULLMASK, incl, o);
        if ((s & 31) >= (uint32_t)o) incl += v;
    }
    if ((s & 31) == 31) sc[s >> 5] = incl;
    __syncthreads();
    if (s < 32) {
        unsigned long long t = sc[s];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long v = __shfl_up_sync(FULLMASK, t, o);
            if (s >= (uint32_t)o) t += v;
        }
        sc[32 + s] = t;  // inclusive prefix of the warp sums
    }
    __syncthreads();
    incl += (s >> 5) ? sc[32 + (s >> 5) - 1] : 0ull;
    const unsigned long long total_items = sc[32 + 31];
    if (s < w.nslots) w.offs[s] = incl - items;
    if (s == 0) {
        w.offs[w.nslots] = total_items;
        w.ctr[C_ACTIVE] = nact;
        w.ctr[C_TOTAL] = (uint32_t)min(total_items, 0xFFFFFFFFull);  // diagnostics
        w.ctr[C_NHEAVY] = 0;
        w.ctr[C_NPULL] = npull;
        if (!w.hnode) {  // profiling counters of the per-slot expansion (k_expand counts edges/cells)
            w.prof[P_ITEMS] += total_items;
            w.prof[P_ENQ] += nenq;
        }
        // joint traversal: size of the union frontier of this level, reset the next one
        w.ctr[C_JQCUR] = w.ctr[C_JQN0 + (l & 1)];
        w.ctr[C_JQN0 + ((l & 1) ^ 1)] = 0;
        w.ctr[C_JHEAVY] = 0;
    }
}

// ====================================================================== expansion (Alg. 1)
template <class RowT> struct Relax {
    bool enq;    // first writer of this row at this level -> next frontier
    bool ident;  // completed the row -> identified at level l+1
    int cells;   // cells turned from inf to l+1 by this thread, + ATOM_ONE if it issued the atomic
};
// relax() reports the atomic it issued as ATOM_ONE in `cells`; the expansion adds the cells to
// a per-lane counter and the atomics, one ballot per unrolled edge, to a warp-uniform counter
// (uniform registers: no pressure on the 32-register budget of the 8-blocks/SM kernels)
constexpr int ATOM_ONE = 1 << 16;
__device__ __forceinline__ void cnt_add(uint32_t &cells_acc, uint32_t &atoms_acc, int cells) {
    cells_acc += cells & 0xFFFF;
    atoms_acc += __popc(__ballot_sync(FULLMASK, cells >= ATOM_ONE));
}

// Relaxation of edge (f -> n) for the byte-columns in `mask` at level l (Alg. 1 lines 12-17),
// given the (possibly stale) row hn read earlier: one atomicAnd writes l+1 into every selected
// byte that is still 0xFF; the old row says whether this thread is the first writer of n's row
// at this level (enqueue) and whether it completed the row (identification at l+1, R10).
template <class RowT>
__device__ __forceinline__ Relax<RowT> relax(const HV<RowT> &H, uint32_t n, RowT hn, RowT mask, uint32_t l) {
    typedef Row<RowT> R;
    Relax<RowT> r{false, false, 0};
    const RowT FF = R::splat(0xFF);
    RowT need = mask & R::eq(hn, FF);
    if (!need) return r;
    RowT andm = ~need | (need & R::splat(l + 1));
    RowT old = R::atomic_and(H + n, andm);
    const RowT oldFF = R::eq(old, FF);
    RowT changed = need & oldFF;
    r.cells = ATOM_ONE;
    if (!changed) return r;
    r.cells += R::ones(changed);
    r.enq = R::eq(old, R::splat(l + 1)) == 0;  // no cell of n was written at this level before
    r.ident = (oldFF & ~need) == 0;            // this write completed the row: every inf cell was in need
    return r;
}

// The same relaxation for U edges of one lane at once: every atomic is issued before any of
// their results is used, so a lane has U atomics in flight instead of one (ncu r02e: the
// instructions after each atomicAnd carried the top stall samples).  EXP_BATCH_ATOM=0 keeps
// the one-at-a-time relax() (A/B).
#ifndef EXP_BATCH_ATOM
#define EXP_BATCH_ATOM 0  // measured: -1.5 % at C2, equal at C5 (r02h A/B)
#endif
template <class RowT, int U>
__device__ __forceinline__ void relax_n(RowT *const (&row)[U], const RowT (&hn)[U], const RowT (&mask)[U],
                                        const bool (&ev)[U], uint32_t l, bool (&enq)[U], bool (&idn)[U],
                                        uint32_t &cells) {  // (A/B variant: atomics not counted)
    typedef Row<RowT> R;
    const RowT FF = R::splat(0xFF), L1 = R::splat(l + 1);
    RowT need[U], andm[U], old[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
        need[u] = ev[u] ? mask[u] & R::eq(hn[u], FF) : (RowT)0;
        andm[u] = ~need[u] | (need[u] & L1);
    }
#pragma unroll
    for (int u = 0; u < U; u++) old[u] = need[u] ? R::atomic_and(row[u], andm[u]) : (RowT)0;
#pragma unroll
    for (int u = 0; u < U; u++) {
        const RowT changed = need[u] & R::eq(old[u], FF);
        cells += R::ones(changed);
        enq[u] = changed && R::eq(old[u], L1) == 0;
        idn[u] = changed && R::eq(old[u] & andm[u], FF) == 0;
    }
}

// Next frontier Q_{l+1}: a node is appended by the first writer of its row at level l (new
// entry) or, if it keeps pending edges (Alg. 1 lines 9-11), by its own item (retained entry,
// tag bit 31).  A retained entry whose row also carries l+1 is a duplicate and is skipped by
// the consumer, so every node of F is expanded exactly once per level without a
// separate flag array: the level stored in H is the frontier flag.
constexpr uint32_t RETAINED = 0x80000000u;
__device__ __forceinline__ void frontier_push(const WsDev &w, bool want, uint32_t s, uint32_t entry, uint32_t nxt) {
    // warp-aggregated append; new (untagged) entries are also counted in st.reached, the
    // visited estimate of the direction-optimising heuristic
    const uint32_t m = __ballot_sync(FULLMASK, want);
    if (!m) return;
    // usually every pushing lane is in one slot (items are slot-contiguous): no match_any
    const uint32_t s0 = __shfl_sync(FULLMASK, s, __ffs(m) - 1);
    if (__all_sync(FULLMASK, !want || s == s0)) {
        const uint32_t leader = __ffs(m) - 1;
        uint32_t base = 0;
        if (lane_id() == leader) {
            base = atomicAdd(&w.st[s0].nq[nxt], __popc(m));
            if (w.track_reached && !(entry & RETAINED)) atomicAdd(&w.st[s0].reached, __popc(m));
        }
        base = __shfl_sync(FULLMASK, base, leader);
        if (base + __popc(m) > w.qcap) {  // more entries than the queue holds: flag, retry bigger
            if (lane_id() == leader) atomicOr(&w.st[s0].err, (uint32_t)E_QUEUE);
            return;
        }
        if (want) w.Q(s0, nxt)[base + __popc(m & lanemask_lt())] = entry;
        return;
    }
    if (want) {
        uint32_t peers = __match_any_sync(m, s);
        uint32_t leader = __ffs(peers) - 1;
        uint32_t rank = __popc(peers & lanemask_lt());
        uint32_t base = 0;
        if (lane_id() == leader) {
            base = atomicAdd(&w.st[s].nq[nxt], __popc(peers));
            if (w.track_reached && !(entry & RETAINED)) atomicAdd(&w.st[s].reached, __popc(peers));
        }
        base = __shfl_sync(peers, base, leader);
        if (base + __popc(peers) > w.qcap) {
            if (lane_id() == leader) atomicOr(&w.st[s].err, (uint32_t)E_QUEUE);
        } else {
            w.Q(s, nxt)[base + rank] = entry;
        }
    }
}

// U pushes per lane at once (the unrolled edges of one chunk, after NR leading retained
// entries): when every pushing (lane, u) is in one slot, a single queue-counter atomic
// covers them all.
// su: the warp-uniform slot of every push when the caller knows it (all of the warp's items in
// one slot), else EMPTY (then the slots are compared).
template <int U, int NR = 0>
__device__ __forceinline__ void frontier_push_n(const WsDev &w, const bool (&want)[U], const uint32_t (&s)[U],
                                                const uint32_t (&entry)[U], uint32_t nxt, uint32_t su = EMPTY) {
    uint32_t m[U], any = 0;
#pragma unroll
    for (int u = 0; u < U; u++) any |= (m[u] = __ballot_sync(FULLMASK, want[u]));
    if (!any) return;
    uint32_t s0 = su;
    bool ok = true;
    if (su == EMPTY) {
        int u0 = 0;
#pragma unroll
        for (int u = U - 1; u >= 0; u--)
            if (m[u]) u0 = u;
#pragma unroll
        for (int u = 0; u < U; u++)
            if (u == u0) s0 = __shfl_sync(FULLMASK, s[u], __ffs(m[u]) - 1);
#pragma unroll
        for (int u = 0; u < U; u++) ok &= !want[u] || s[u] == s0;
    }
    if (__all_sync(FULLMASK, ok)) {
        uint32_t cnt = 0;
#pragma unroll
        for (int u = 0; u < U; u++) cnt += __popc(m[u]);
        uint32_t base = 0;
        if (lane_id() == 0) {
            base = atomicAdd(&w.st[s0].nq[nxt], cnt);
            uint32_t fresh = cnt;  // new (untagged) entries feed the visited estimate
#pragma unroll
            for (int u = 0; u < NR; u++) fresh -= __popc(m[u]);
            if (w.track_reached && fresh) atomicAdd(&w.st[s0].reached, fresh);
        }
        base = __shfl_sync(FULLMASK, base, 0);
        if (base + cnt > w.qcap) {
            if (lane_id() == 0) atomicOr(&w.st[s0].err, (uint32_t)E_QUEUE);
            return;
        }
        uint32_t *Qd = w.Q(s0, nxt);
        const uint32_t lt = lanemask_lt();
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (m[u]) {  // warp-uniform: most unrolled edges push nothing
                if (want[u]) Qd[base + __popc(m[u] & lt)] = entry[u];
                base += __popc(m[u]);
            }
        }
        return;
    }
#pragma unroll
    for (int u = 0; u < U; u++) frontier_push(w, want[u], s[u], entry[u], nxt);
}

__device__ __forceinline__ void cand_push(const GraphDev &g, const WsDev &w, bool want, uint32_t s, uint32_t n,
                                          uint32_t level) {
    uint32_t pos = warp_append(want, s, &w.st[0].ncand, sizeof(SlotState) / 4);
    if (want) {  // key (S^c, caller id): the (S^c, v) order of R13/R23 uses the caller's ids
        if (pos < w.capc) w.CK(s)[pos] = (uint64_t)level << 32 | __ldg(g.iperm + n);
        else atomicOr(&w.st[s].err, (uint32_t)E_CAND);
    }
}

__device__ __forceinline__ uint32_t upper_bound_act(const uint8_t *act, uint32_t lo, uint32_t hi, uint32_t l) {
    while (lo < hi) {  // first index with act > l
        uint32_t m = (lo + hi) >> 1;
        if (__ldg(act + m) <= l) lo = m + 1; else hi = m;
    }
    return lo;
}
__device__ __forceinline__ uint32_t lower_bound_act(const uint8_t *act, uint32_t lo, uint32_t hi, uint32_t l) {
    while (lo < hi) {  // first index with act >= l
        uint32_t m = (lo + hi) >> 1;
        if (__ldg(act + m) < l) lo = m + 1; else hi = m;
    }
    return lo;
}

// Gate ranges of out-row d at level l (activation-sorted row [rb, re)): hi = first edge with
// a > l, eqlo = first edge with a >= l.  Rows <= 8 edges: byte-SIMD over the packed
// activations in the descriptor; longer rows: the gate offset table (two loads, one line),
// binary search only past AOFF_LEVELS.
__device__ __forceinline__ void gate_range_t(const uint8_t *act, const uint32_t *aoff, const uint4 &d, uint32_t l,
                                             uint32_t &hi, uint32_t &eqlo) {
    const uint32_t rb = d.x, re = d.x + d.y;
    if (d.y <= 8) {  // padding 0xFF never passes the gate
        const uint32_t L4 = l * 0x01010101u;
        hi = rb + ((__popc(__vcmpleu4(d.z, L4)) + __popc(__vcmpleu4(d.w, L4))) >> 3);
        eqlo = rb + ((__popc(__vcmpltu4(d.z, L4)) + __popc(__vcmpltu4(d.w, L4))) >> 3);
    } else if (l < AOFF_LEVELS) {
        const uint32_t *t = aoff + (size_t)d.z * AOFF_LEVELS;
        hi = __ldg(t + l);
        eqlo = l ? __ldg(t + l - 1) : rb;
    } else {
        const uint32_t b = __ldg(aoff + (size_t)d.z * AOFF_LEVELS + AOFF_LEVELS - 1);
        hi = upper_bound_act(act, b, re, l);
        eqlo = lower_bound_act(act, b, hi, l);
    }
}
__device__ __forceinline__ void gate_range(const GraphDev &g, const uint4 &d, uint32_t l, uint32_t &hi, uint32_t &eqlo) {
    gate_range_t(g.act, g.aoff, d, l, hi, eqlo);
}
__device__ __forceinline__ void gate_range_in(const GraphDev &g, const uint4 &d, uint32_t l, uint32_t &hi, uint32_t &eqlo) {
    gate_range_t(g.iact, g.iaoff, d, l, hi, eqlo);
}

// Work item = one frontier node of one slot.  Each warp takes 32 items: lane i does the
// per-node part (row bounds, CF check, retention, activation range by binary search in the
// activation-sorted row), then the warp walks the concatenated active ranges edge-parallel,
// three edges in flight per lane (measured: 2 -1.2 %, 4 -1..-3 % from spills).
#ifndef EXP_UNROLL
#define EXP_UNROLL 3
#endif
#ifndef EXP_SMALL
#define EXP_SMALL 0  // >0: ranges of at most this many due edges walked lane-locally (4: -10 % at C2, -3 % at C5; r02n)
#endif
#ifndef EXP_MINB
#define EXP_MINB 8  // 32 registers (7 blocks would give the same 32: allocation is in units of 8)
#endif
// 64-bit rows (5-8 keywords) need more registers: at 8 blocks (32 registers) the u64 loop
// spills to local memory in its hot path (ncu r02e: LDL + short-scoreboard stalls).
#ifndef EXP_MINB64
#define EXP_MINB64 6
#endif
// BIG: graphs of >= EXP_BIG_V nodes, whose expansion waits on random HBM rows rather than on
// issue: 4 blocks/SM (no spills) for every row width -- fewer warps in flight thrash L2 less
// (measured against 8/6 blocks: +5-8 % at config 5, +13 % at config 3; -6 % at config 2 if
// used there; profiles/r02_ab_experiments.txt r02x-r02ab)
#ifndef EXP_BIG_V
#define EXP_BIG_V (4u << 20)
#endif
#ifndef EXP_MINB_BIG
#define EXP_MINB_BIG 4
#endif
#ifndef EXP_MINB64_BIG
#define EXP_MINB64_BIG 4
#endif
#ifndef EXP_UNROLL_BIG
#define EXP_UNROLL_BIG 3
#endif
#ifndef HEAVY_UNROLL_BIG
#define HEAVY_UNROLL_BIG 2
#endif
template <class RowT, bool BIG = false> struct ExpMinB {
    static constexpr int v = BIG ? (sizeof(RowT) == 8 ? EXP_MINB64_BIG : EXP_MINB_BIG)
                                 : (sizeof(RowT) == 8 ? EXP_MINB64 : EXP_MINB);
};
// Item fields of one non-empty active range, compacted per warp in shared memory for the
// edge walk: edge index e = delta + idx, and edges with idx >= thr also carry the old columns.
template <class RowT> struct alignas(16) OwnF {
    uint32_t delta, thr, s;
    RowT nw, od;
};

// Vertex-partitioned push: a rank walks the out-edges of the
// frontier nodes it owns, [lo, hi), and instead of writing H it ORs each newly reachable
// cell (n, j) into bit plane j of n's OWNER's exchange slice -- xs[owner] is that slice, in
// peer memory over NVLink in a real multi-rank run (the fused exchange), or a region of one
// buffer for simulated partitions.  Slice layout [pull position][plane][wc words] over the
// owner's range.  H stays as it was at the start of the level on every rank until
// k_vp_apply_words writes the all-gathered planes.  The item phase (relaxation counts,
// retained entries) runs on every rank for every item (`side`), so the frontier queues, the
// counts and the candidates are replicated without another collective.
struct VpPush {
    uint32_t lo, hi;          // this launch's owned source range
    uint32_t nranks, wc, side;
    const uint32_t *bounds;   // nranks + 1 owner bounds (multiples of 32)
    uint32_t *const *xs;      // per owner: its exchange slice for this level
};
template <class RowT>
__device__ __forceinline__ void vp_mark(const VpPush &vp, uint32_t p, uint32_t n, RowT need) {
    constexpr uint32_t RB = sizeof(RowT);
    uint32_t r = 0;
    while (r + 1 < vp.nranks && n >= __ldg(vp.bounds + r + 1)) r++;
    const uint32_t i = n - __ldg(vp.bounds + r);
    uint32_t *x = vp.xs[r] + (size_t)p * RB * vp.wc + (i >> 5);
#pragma unroll
    for (uint32_t j = 0; j < RB; j++)
        if ((need >> (8 * j)) & 0xFF) atomicOr(x + (size_t)j * vp.wc, 1u << (i & 31));
}

// WIDE: 64-bit frontier-item indices, for batches whose level can exceed 2^32 items
// (slots x queue capacity >= 2^32, e.g. 200 queries on a 30M-node graph); the common
// case keeps the 32-bit loop.  VPX: the vertex-partitioned push (VpPush above).
// CNT: count the relaxation atomics (riki_stats.exp_atomics) -- the profiling-mode variant (the
// per-edge ballot costs ~2 % at config 2, so the production path does not count them).
template <class RowT, bool WIDE, bool VPX = false, bool CNT = false, bool BIG = false>
__global__ void __launch_bounds__(256, (ExpMinB<RowT, BIG>::v)) k_expand(GraphDev g, WsDev w, int ph, uint32_t l_arg,
                                                                  VpPush vp = VpPush{}) {
    constexpr int UNR = BIG ? EXP_UNROLL_BIG : EXP_UNROLL;
    typedef Row<RowT> R;
    const uint32_t l = l_arg == LV_DEVICE ? w.ctr[C_LEVEL] : l_arg;
    typedef typename std::conditional<WIDE, unsigned long long, uint32_t>::type IdxT;
    __shared__ IdxT s_offs[MAX_SLOTS + 1];
    __shared__ uint32_t s_info[MAX_SLOTS];
    __shared__ OwnF<RowT> s_own[8][32];
    const uint32_t ns = w.nslots;
    for (uint32_t i = threadIdx.x; i <= ns; i += blockDim.x) s_offs[i] = (IdxT)w.offs[i];
    for (uint32_t i = threadIdx.x; i < ns; i += blockDim.x) {
        const SlotState &st = w.st[i];
        s_info[i] = st.blocking | st.collect << 1 | st.pull << 2 | st.T[ph] << 8;
    }
    __syncthreads();
    const IdxT total = s_offs[ns];
    const uint32_t lane = lane_id();
    const uint32_t cur = l & 1, nxt = cur ^ 1;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const RowT L = R::splat(l);
    RowT *const Hb = (RowT *)w.H[ph];  // per-slot layout (HGRP groups; never joint here)
    const size_t V = w.V;
    OwnF<RowT> *const own = s_own[threadIdx.x >> 5];
    uint32_t p_edges = 0, p_cells = 0, p_work = 0, p_atoms = 0;  // items and queue entries: k_plan

    for (IdxT base = (IdxT)gw * 32; base < total; base += (IdxT)nw * 32) {
        const IdxT item = base + lane;
        bool valid = item < total;
        // slots of this warp's 32 items: two warp-uniform searches, then (rarely) a short
        // per-lane search between them
        const uint32_t sA = find_slot_warp(s_offs, ns, base);
        const uint32_t sB = find_slot_warp(s_offs, ns, min(base + 31, total - 1));
        uint32_t s = sA, f = 0, lo = 0, len = 0, relaxn = 0, eq0 = 0;
        RowT newc = 0, oldc = 0;
        bool retain = false;
        if (valid) {
            if (sB != sA) s = find_slot(s_offs + sA, sB - sA + 1, item) + sA;
            uint32_t info = s_info[s];
            uint32_t ent = STREAM_LD(w.Q(s, cur) + (uint32_t)(item - s_offs[s]));
            f = ent & ~RETAINED;
            RowT Rf = R::load(Hb + ((size_t)(s / HGRP) * V + f) * HGRP + s % HGRP);
            const uint4 d = __ldg(g.desc + f);  // issued with the row load (dropped if dup / blocked)
            RowT used = used_mask<RowT>(info >> 8);
            bool dup = (ent & RETAINED) && (R::eq(Rf, L) & used);
            bool blocked = (info & 1) && R::le(Rf, L) == (RowT)~(RowT)0;  // CF: row complete, max <= l
#if EXP_STATS
            if (dup) atomicAdd(&w.prof[P_X_DUP], 1ull);
            else if (blocked) atomicAdd(&w.prof[P_X_BLOCKED], 1ull);
#endif
            if (!dup && !blocked) {
                newc = R::eq(Rf, L) & used;   // reached at level l (or seeds at l = 0)
                oldc = R::lt(Rf, L) & used;   // reached earlier: only edges with a == l are due now
                const uint32_t rb = d.x, re = d.x + d.y;
                if (re > rb && (newc | oldc)) {
                    uint32_t hi, eqlo;
                    gate_range(g, d, l, hi, eqlo);
                    retain = hi < re;  // Alg. 1 lines 9-11: some a_fn > l keeps f a frontier
                    lo = newc ? rb : eqlo;
                    eq0 = eqlo;
                    len = hi - lo;
                    relaxn = (hi - rb) * R::ones(newc) + (hi - eqlo) * R::ones(oldc);
                    p_work += len > 0;
#if EXP_STATS
                    atomicAdd(&w.prof[len ? P_X_WORK : P_X_IDLE], 1ull);
#endif
                    if (VPX) {
                        if (f < vp.lo || f >= vp.hi) len = 0;  // another rank walks this node's edges
                        if (!vp.side) { relaxn = 0; retain = false; }  // counted and retained once
                    } else if (info & 4) {
                        len = 0;  // pull slot: relaxed bottom-up by k_pull
                    }
                    p_edges += len;
                    if (len > HEAVY) {
                        uint32_t nch = (len + CHUNK - 1) / CHUNK;
                        uint32_t p = atomicAdd(&w.ctr[C_NHEAVY], nch);
                        if (p + nch <= w.heavy_cap) {
                            for (uint32_t c = 0; c < nch; c++)
                                w.heavy[p + c] = make_uint4(s, f, lo + c * CHUNK, min(lo + (c + 1) * CHUNK, hi));
                        } else {
                            atomicOr(&w.st[s].err, (uint32_t)E_HEAVY);
                        }
                        len = 0;
                    }
                }
            }
        }
        {   // relaxation count per slot (aggregated)
            if (sA == sB) {
                uint32_t sum = __reduce_add_sync(FULLMASK, relaxn);
                if (lane == 0 && sum) atomicAdd(&w.st[sA].relax[ph], (unsigned long long)sum);
            } else {
                uint32_t vm = __ballot_sync(FULLMASK, valid);
                if (valid) {
                    uint32_t peers = __match_any_sync(vm, s);
                    uint32_t sum = __reduce_add_sync(peers, relaxn);
                    if (lane == __ffs(peers) - 1 && sum) atomicAdd(&w.st[s].relax[ph], (unsigned long long)sum);
                }
            }
        }
#if EXP_SMALL
        // Short ranges (<= EXP_SMALL due edges, most items on power-law graphs): each lane walks
        // its own range with all its edges in flight, no owner search; the warp-cooperative
        // walk below takes the longer ranges.
        if (!VPX) {
            const bool small = len > 0 && len <= EXP_SMALL;
            if (__any_sync(FULLMASK, small)) {
                uint32_t nn[EXP_SMALL];
                RowT hh[EXP_SMALL], mk[EXP_SMALL];
                bool ev[EXP_SMALL];
#pragma unroll
                for (int u = 0; u < EXP_SMALL; u++) {
                    ev[u] = small && (uint32_t)u < len;
                    nn[u] = ev[u] ? STREAM_LD(g.col + lo + u) : 0;
                    mk[u] = newc | (lo + u >= eq0 ? oldc : (RowT)0);
                }
                RowT *const Hs_ = Hb + (size_t)(s / HGRP) * V * HGRP + s % HGRP;
#pragma unroll
                for (int u = 0; u < EXP_SMALL; u++) hh[u] = ev[u] ? R::load(Hs_ + (size_t)nn[u] * HGRP) : (RowT)0;
                bool pw[EXP_SMALL + 1], idn[EXP_SMALL];
                uint32_t ps[EXP_SMALL + 1], pe[EXP_SMALL + 1];
                pw[0] = retain && small;
                ps[0] = s;
                pe[0] = f | RETAINED;
#pragma unroll
                for (int u = 0; u < EXP_SMALL; u++) {
                    Relax<RowT> r{false, false, 0};
                    if (ev[u]) r = relax<RowT>(HV<RowT>{Hs_, (uint32_t)HGRP}, nn[u], hh[u], mk[u], l);
                    if (CNT) cnt_add(p_cells, p_atoms, r.cells);
                    else p_cells += r.cells & 0xFFFF;
                    pw[u + 1] = r.enq;
                    ps[u + 1] = s;
                    pe[u + 1] = nn[u];
                    idn[u] = r.ident;
                }
                frontier_push_n<EXP_SMALL + 1, 1>(w, pw, ps, pe, nxt);
                bool anyid = false;
#pragma unroll
                for (int u = 0; u < EXP_SMALL; u++) anyid |= idn[u];
                if (__any_sync(FULLMASK, anyid)) {
                    const bool coll = (s_info[s] >> 1) & 1;
#pragma unroll
                    for (int u = 0; u < EXP_SMALL; u++) cand_push(g, w, idn[u] && coll, s, nn[u], l + 1);
                }
                if (small) { retain = false; len = 0; }
            }
        }
#endif
        // Edge-parallel walk over the concatenated active ranges, UNR (EXP_UNROLL, EXP_UNROLL_BIG) edges per lane in
        // flight.  The non-empty ranges are compacted into s_own (rank order = start order);
        // the owner of edge position p of a 32-wide chunk is found from the bit mask of range
        // starts inside the chunk (one OR-reduction) instead of a per-edge binary search.
        const uint32_t incl = warp_incl_scan(len);
        const uint32_t tot = __shfl_sync(FULLMASK, incl, 31);
        if (tot == 0) {
            frontier_push(w, retain, s, f | RETAINED, nxt);
            continue;
        }  // otherwise the retained entries go out with the first chunk's pushes
        const uint32_t excl = incl - len;
        {
            const uint32_t NE = __ballot_sync(FULLMASK, len > 0);
            __syncwarp();  // previous iteration's readers are done with s_own
            if (len > 0) {
                OwnF<RowT> o;
                o.delta = lo - excl;
                o.thr = eq0 - lo + excl;
                o.s = s;
                o.nw = newc;
                o.od = oldc;
                own[__popc(NE & lanemask_lt())] = o;
            }
            __syncwarp();
        }
        const uint32_t le_mask = lanemask_lt() | (1u << lane);
        int own_last = -1;
        for (uint32_t eb = 0; eb < tot; eb += 32 * UNR) {
            uint32_t n[UNR], o_s[UNR];
            RowT mask[UNR], hn[UNR];
            bool ev[UNR];
#pragma unroll
            for (int u = 0; u < UNR; u++) {
                const uint32_t cb = eb + 32 * u;
                const uint32_t off = excl - cb;  // < 32 iff this lane's range starts in the chunk
                const uint32_t M = __reduce_or_sync(FULLMASK, (len > 0 && off < 32) ? 1u << off : 0u);
                const int own0 = own_last + (int)(M & 1u);
                const int ow = own0 + __popc(M & ~1u & le_mask);
                own_last = own0 + __popc(M & ~1u);
                const uint32_t idx = cb + lane;
                ev[u] = idx < tot;
                const OwnF<RowT> o = own[ev[u] ? ow : 0];
                o_s[u] = o.s;
                n[u] = ev[u] ? STREAM_LD(g.col + (uint32_t)(o.delta + idx)) : 0;  // delta wraps: add in 32 bits
                mask[u] = o.nw | (idx >= o.thr ? o.od : (RowT)0);  // [eqlo, hi) are the edges with a == l
            }
#pragma unroll
            for (int u = 0; u < UNR; u++)
                hn[u] = ev[u] ? R::load(Hb + ((size_t)(o_s[u] / HGRP) * V + n[u]) * HGRP + o_s[u] % HGRP) : (RowT)0;
            bool enq[UNR], idn[UNR];
            if (!VPX && EXP_BATCH_ATOM) {
                RowT *rowp[UNR];
#pragma unroll
                for (int u = 0; u < UNR; u++)
                    rowp[u] = Hb + ((size_t)(o_s[u] / HGRP) * V + n[u]) * HGRP + o_s[u] % HGRP;
                relax_n<RowT, UNR>(rowp, hn, mask, ev, l, enq, idn, p_cells);
            } else {
#pragma unroll
                for (int u = 0; u < UNR; u++) {
                    Relax<RowT> r{false, false, 0};
                    if (VPX) {  // H is read-only during a partitioned level: mark the owner's bit planes
                        const RowT need = mask[u] & R::eq(hn[u], R::splat(0xFF));
                        if (ev[u] && need) vp_mark<RowT>(vp, w.ppos[o_s[u]], n[u], need);
                    } else if (ev[u]) {
                        r = relax<RowT>(HV<RowT>{Hb + (size_t)(o_s[u] / HGRP) * V * HGRP + o_s[u] % HGRP, (uint32_t)HGRP},
                                        n[u], hn[u], mask[u], l);
                    }
                    if (CNT) cnt_add(p_cells, p_atoms, r.cells);
                    else p_cells += r.cells & 0xFFFF;
                    enq[u] = r.enq;
                    idn[u] = r.ident;
                }
            }
            {
                bool pw[UNR + 1];
                uint32_t ps[UNR + 1], pe[UNR + 1];
                pw[0] = retain;
                ps[0] = s;
                pe[0] = f | RETAINED;
#pragma unroll
                for (int u = 0; u < UNR; u++) {
                    pw[u + 1] = enq[u];
                    ps[u + 1] = o_s[u];
                    pe[u + 1] = n[u];
                }
                frontier_push_n<UNR + 1, 1>(w, pw, ps, pe, nxt, sA == sB ? sA : EMPTY);
                retain = false;
            }
            {   // identification appends: skipped (one vote) when no lane completed a row
                bool anyid = false;
#pragma unroll
                for (int u = 0; u < UNR; u++) anyid |= idn[u];
                if (__any_sync(FULLMASK, anyid)) {
#pragma unroll
                    for (int u = 0; u < UNR; u++)
                        cand_push(g, w, idn[u] && ((s_info[o_s[u]] >> 1) & 1), o_s[u], n[u], l + 1);
                }
            }
        }
    }
    p_edges = warp_sum(p_edges);
    p_cells = warp_sum(p_cells);
    p_work = warp_sum(p_work);
    if (lane == 0 && (p_edges | p_cells | p_atoms)) {
        atomicAdd(&w.prof[P_EDGES], (unsigned long long)p_edges);
        atomicAdd(&w.prof[P_NEWCELLS], (unsigned long long)p_cells);
        atomicAdd(&w.prof[P_ATOMS], (unsigned long long)p_atoms);  // warp total already
        atomicAdd(&w.prof[P_ITEMS_WORK], (unsigned long long)p_work);
    }
}

// Heavy ranges (hub rows): one warp per CHUNK-edge piece, HEAVY_UNROLL edges per lane in flight.
#ifndef HEAVY_UNROLL
#define HEAVY_UNROLL 2
#endif
template <class RowT, bool VPX = false, bool CNT = false, bool BIG = false>
__global__ void __launch_bounds__(256, (ExpMinB<RowT, BIG>::v)) k_expand_heavy(GraphDev g, WsDev w, int ph, uint32_t l_arg,
                                                                       VpPush vp = VpPush{}) {
    constexpr int HUNR = BIG ? HEAVY_UNROLL_BIG : HEAVY_UNROLL;
    const uint32_t l = l_arg == LV_DEVICE ? w.ctr[C_LEVEL] : l_arg;
    typedef Row<RowT> R;
    const uint32_t lane = lane_id();
    const uint32_t nxt = (l & 1) ^ 1;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    uint32_t nh = min(w.ctr[C_NHEAVY], w.heavy_cap);
    const RowT L = R::splat(l);
    uint32_t p_cells = 0, p_atoms = 0;  // p_atoms: warp total (cnt_add)
    for (uint32_t it = gw; it < nh; it += nw) {
        uint4 h = w.heavy[it];
        uint32_t s = h.x;
        // after an overflow (E_HEAVY, fatal) entries past the last write are stale: stay in bounds
        if (s >= w.nslots || h.y >= w.V || h.z > h.w || h.w > g.E) continue;
        const SlotState &st = w.st[s];
        RowT used = used_mask<RowT>(st.T[ph]);
        const HV<RowT> Hs = w.Hs<RowT>(ph, s);  // per-slot layout (never joint here)
        RowT Rf = R::load(Hs + h.y);  // values <= l are final; concurrent l+1 writes don't change the masks
        RowT newc = R::eq(Rf, L) & used, oldc = R::lt(Rf, L) & used;
        bool collect = st.collect;
        for (uint32_t e0 = h.z; e0 < h.w; e0 += 32 * HUNR) {
            uint32_t n[HUNR], a[HUNR];
            RowT hn[HUNR];
#pragma unroll
            for (int u = 0; u < HUNR; u++) {
                uint32_t e = e0 + 32 * u + lane;
                n[u] = e < h.w ? STREAM_LD(g.col + e) : 0;
                a[u] = e < h.w ? __ldg(g.act + e) : 0xFF;
            }
#pragma unroll
            for (int u = 0; u < HUNR; u++) hn[u] = (e0 + 32 * u + lane < h.w) ? R::load(Hs + n[u]) : (RowT)0;
            bool enq[HUNR], idn[HUNR];
            uint32_t ss[HUNR];
#pragma unroll
            for (int u = 0; u < HUNR; u++) ss[u] = s;
            if (!VPX && EXP_BATCH_ATOM) {
                RowT *rowp[HUNR], mk[HUNR];
                bool ev[HUNR];
#pragma unroll
                for (int u = 0; u < HUNR; u++) {
                    ev[u] = e0 + 32 * u + lane < h.w;
                    rowp[u] = Hs + n[u];
                    mk[u] = newc | (a[u] == l ? oldc : (RowT)0);
                }
                relax_n<RowT, HUNR>(rowp, hn, mk, ev, l, enq, idn, p_cells);
            } else
#pragma unroll
            for (int u = 0; u < HUNR; u++) {
                Relax<RowT> r{false, false, 0};
                if (e0 + 32 * u + lane < h.w) {
                    RowT mask = newc | (a[u] == l ? oldc : (RowT)0);
                    if (VPX) {
                        const RowT need = mask & R::eq(hn[u], R::splat(0xFF));
                        if (need) vp_mark<RowT>(vp, w.ppos[s], n[u], need);
                    } else {
                        r = relax<RowT>(Hs, n[u], hn[u], mask, l);
                    }
                }
                if (CNT) cnt_add(p_cells, p_atoms, r.cells);
                else p_cells += r.cells & 0xFFFF;
                enq[u] = r.enq;
                idn[u] = r.ident;
            }
            frontier_push_n<HUNR>(w, enq, ss, n, nxt, s);  // one chunk: one slot
            bool anyid = false;
#pragma unroll
            for (int u = 0; u < HUNR; u++) anyid |= idn[u] && collect;
            if (__any_sync(FULLMASK, anyid))
#pragma unroll
                for (int u = 0; u < HUNR; u++) cand_push(g, w, idn[u] && collect, s, n[u], l + 1);
        }
    }
    p_cells = warp_sum(p_cells);
    if (lane == 0 && (p_cells | p_atoms)) {
        atomicAdd(&w.prof[P_NEWCELLS], (unsigned long long)p_cells);
        atomicAdd(&w.prof[P_ATOMS], (unsigned long long)p_atoms);
    }
}

// Vertex-partitioned exchange slice: bit plane j of pull slot p holds, for each node of the
// rank's range (offset i), whether column j was reached at level l + 1.
template <class RowT>
__device__ __forceinline__ void vp_set_bits(uint32_t *x, uint32_t p, uint32_t wc, uint32_t i, RowT found) {
    constexpr uint32_t RB = sizeof(RowT);
#pragma unroll
    for (uint32_t j = 0; j < RB; j++)
        if ((found >> (8 * j)) & 0xFF) atomicOr(x + ((size_t)p * RB + j) * wc + (i >> 5), 1u << (i & 31));
}

// Vertex-partitioned mode, after the all-gather: every rank applies every rank's slice to its
// replicated H (identical H, blocks, frontiers and candidates on all ranks), with the same
// write, next-frontier append and identification at l + 1 as the single-GPU pull.  Thread
// per (rank, node offset); x = [rank][pull slot][plane][wc].
template <class RowT>
__global__ void __launch_bounds__(256) k_vp_apply(GraphDev g, WsDev w, int ph, uint32_t l, const uint32_t *x,
                                                  uint32_t wc, uint32_t nranks, const uint32_t *bounds, uint32_t npull) {
    typedef Row<RowT> R;
    constexpr uint32_t RB = sizeof(RowT);
    const uint32_t p = blockIdx.y, s = w.pslots[p];
    const HV<RowT> H = w.Hs<RowT>(ph, s);
    const bool collect = w.st[s].collect;
    const uint32_t nxt = (l & 1) ^ 1;
    const size_t chunk = (size_t)npull * RB * wc;
    const uint64_t total = (uint64_t)nranks * wc * 32;
    uint32_t p_cells = 0;
    for (uint64_t b = (uint64_t)blockIdx.x * blockDim.x; b < total; b += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t = b + threadIdx.x;
        bool enq = false, id = false;
        uint32_t n = 0;
        if (t < total) {
            const uint32_t r = (uint32_t)(t / ((uint64_t)wc * 32)), i = (uint32_t)(t % ((uint64_t)wc * 32));
            n = __ldg(bounds + r) + i;
            if (n < __ldg(bounds + r + 1)) {
                const uint32_t *xs = x + r * chunk + (size_t)p * RB * wc + (i >> 5);
                RowT found = 0;
#pragma unroll
                for (uint32_t j = 0; j < RB; j++)
                    if ((__ldg(xs + (size_t)j * wc) >> (i & 31)) & 1u) found |= (RowT)0xFF << (8 * j);
                if (found) {
                    const RowT Rn = R::load(H + n);
                    const RowT nr = (Rn & ~found) | (found & R::splat(l + 1));
                    *(H + n) = nr;
                    enq = true;
                    id = collect && R::eq(nr, R::splat(0xFF)) == 0;
                    p_cells += R::ones(found);
                }
            }
        }
        frontier_push(w, enq, s, n, nxt);
        cand_push(g, w, id, s, n, l + 1);
    }
    p_cells = warp_sum(p_cells);
    if (lane_id() == 0 && p_cells) atomicAdd(&w.prof[P_NEWCELLS], (unsigned long long)p_cells);
}

// Vertex-partitioned push, after the exchange: the planes of every rank's slice are applied
// to the replicated H on every rank (H, next frontier and identification at l + 1 identical
// everywhere).  Thread per 32-node word of a slice: warps whose words are all zero skip;
// otherwise a warp-uniform loop over the 32 bit positions (frontier_push / cand_push are
// warp collectives).  x: slice r of pull position p, plane j at x + r*stride + (p*RB + j)*wc.
template <class RowT>
__global__ void __launch_bounds__(256) k_vp_apply_words(GraphDev g, WsDev w, int ph, uint32_t l, const uint32_t *x,
                                                        size_t stride, uint32_t wc, uint32_t nranks,
                                                        const uint32_t *bounds) {
    typedef Row<RowT> R;
    constexpr uint32_t RB = sizeof(RowT);
    const uint32_t p = blockIdx.y, s = w.pslots[p];
    const HV<RowT> H = w.Hs<RowT>(ph, s);
    const bool collect = w.st[s].collect;
    const uint32_t nxt = (l & 1) ^ 1;
    const uint32_t total = nranks * wc;
    uint32_t p_cells = 0;
    for (uint32_t b = blockIdx.x * blockDim.x; b < total; b += gridDim.x * blockDim.x) {
        const uint32_t t = b + threadIdx.x;
        uint32_t pl[RB], any = 0, base = 0;
        if (t < total) {
            const uint32_t r = t / wc, wi = t % wc;
            const uint32_t *xs = x + r * stride + (size_t)p * RB * wc + wi;
#pragma unroll
            for (uint32_t j = 0; j < RB; j++) any |= (pl[j] = __ldg(xs + (size_t)j * wc));
            base = __ldg(bounds + r) + wi * 32;
        } else {
#pragma unroll
            for (uint32_t j = 0; j < RB; j++) pl[j] = 0;
        }
        if (!__any_sync(FULLMASK, any != 0)) continue;
        for (uint32_t bit = 0; bit < 32; bit++) {
            bool enq = false, id = false;
            const uint32_t n = base + bit;
            if ((any >> bit) & 1u) {
                RowT found = 0;
#pragma unroll
                for (uint32_t j = 0; j < RB; j++)
                    if ((pl[j] >> bit) & 1u) found |= (RowT)0xFF << (8 * j);
                const RowT Rn = R::load(H + n);  // found cells were infinite at the level start on every rank
                const RowT nr = (Rn & ~found) | (found & R::splat(l + 1));
                *(H + n) = nr;
                enq = true;
                id = collect && R::eq(nr, R::splat(0xFF)) == 0;
                p_cells += R::ones(found);
            }
            frontier_push(w, enq, s, n, nxt);
            cand_push(g, w, id, s, n, l + 1);
        }
    }
    p_cells = warp_sum(p_cells);
    if (lane_id() == 0 && p_cells) atomicAdd(&w.prof[P_NEWCELLS], (unsigned long long)p_cells);
}

// Bottom-up expansion of a dense level (direction-optimising BFS).  Node n with an infinite
// column j takes h_nj = l + 1 iff some in-edge (f -> n) has a <= l, h_fj <= l and f is not
// blocked at l.  This is exactly Alg. 1's push at level l: an unblocked f with
// max(h_fj, a) < l would have relaxed the edge at an earlier level already.  Only n's own
// thread writes its row (no atomics); in-rows are activation-sorted so the scan stops at
// a > l, and as soon as every infinite column found a parent.  Heavy in-rows (internal ids
// < Vh) are scanned by a warp, the rest by one thread each.
//
// Vertex-partitioned mode (vpx != nullptr): only nodes of [lo, hi) are pulled (the in-edges
// this rank owns) and a node's new columns are not written to H but set in bit plane j of
// the rank's exchange slice, vpx[(pull slot * RB + j) * wc + (n - lo) / 32]; k_vp_apply
// writes them on every rank after the all-gather.
template <class RowT> __global__ void __launch_bounds__(256, EXP_MINB) k_pull(GraphDev g, WsDev w, int ph, uint32_t l,
                                                                             uint32_t nbh, uint32_t lo, uint32_t hi,
                                                                             uint32_t *vpx, uint32_t wc) {
    typedef Row<RowT> R;
    const uint32_t s = w.pslots[blockIdx.y];
    const SlotState &st = w.st[s];
    const HV<RowT> H = w.Hs<RowT>(ph, s);
    const RowT used = used_mask<RowT>(st.T[ph]);
    const RowT FF = R::splat(0xFF), L = R::splat(l);
    const bool blocking = st.blocking, collect = st.collect;
    const uint32_t nxt = (l & 1) ^ 1, lane = lane_id();
    uint32_t p_nodes = 0, p_edges = 0, p_cells = 0;
    if (blockIdx.x < nbh) {  // warp per heavy node
        const uint32_t nw = nbh * (blockDim.x >> 5), hh = min(hi, g.Vh);
        for (uint32_t n = lo + blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); n < hh; n += nw) {
            RowT Rn = R::load(H + n);
            RowT inf = R::eq(Rn, FF) & used;
            RowT found = 0;
            if (inf) {
                p_nodes++;
                uint32_t rb = __ldg(g.irow + n), re = __ldg(g.irow + n + 1);
                for (uint32_t k0 = rb; k0 < re; k0 += 32) {
                    uint32_t k = k0 + lane;
                    uint32_t a = k < re ? __ldg(g.iact + k) : 0xFFu;
                    RowT q = 0;
                    if (a <= l) {
                        RowT Rf = R::load(H + __ldg(g.isrc + k));
                        RowT le = R::le(Rf, L);
                        if (!(blocking && le == (RowT)~(RowT)0)) q = le & inf;
                    }
                    p_edges += (a <= l);
                    if constexpr (sizeof(RowT) == 8) {
                        found |= (RowT)__reduce_or_sync(FULLMASK, (uint32_t)q) |
                                 ((RowT)__reduce_or_sync(FULLMASK, (uint32_t)((uint64_t)q >> 32)) << 32);
                    } else {
                        found |= (RowT)__reduce_or_sync(FULLMASK, (uint32_t)q);
                    }
                    if (found == inf || __shfl_sync(FULLMASK, a, 31) > l) break;
                }
            }
            bool enq = false, id = false;
            if (found && lane == 0) {
                if (vpx) {
                    vp_set_bits<RowT>(vpx, blockIdx.y, wc, n - lo, found);
                } else {
                    RowT nr = (Rn & ~found) | (found & R::splat(l + 1));
                    *(H + n) = nr;
                    enq = true;
                    id = collect && R::eq(nr, FF) == 0;
                    p_cells += R::ones(found);
                }
            }
            frontier_push(w, enq, s, n, nxt);
            cand_push(g, w, id, s, n, l + 1);
        }
    } else {  // thread per light node
        const uint32_t stride = (gridDim.x - nbh) * blockDim.x;
        for (uint32_t n0 = max(lo, g.Vh) + (blockIdx.x - nbh) * blockDim.x; n0 < hi; n0 += stride) {
            uint32_t n = n0 + threadIdx.x;
            bool enq = false, id = false;
            if (n < hi) {
                RowT Rn = R::load(H + n);
                RowT inf = R::eq(Rn, FF) & used;
                if (inf) {
                    p_nodes++;
                    RowT found = 0;
                    uint32_t rb = __ldg(g.irow + n), re = __ldg(g.irow + n + 1);
                    for (uint32_t k0 = rb; k0 < re && found != inf; k0 += 4) {
                        uint32_t f[4];
                        bool ok[4];
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            uint32_t k = k0 + u;
                            ok[u] = k < re && __ldg(g.iact + k) <= l;
                            f[u] = ok[u] ? __ldg(g.isrc + k) : 0;
                        }
                        RowT Rf[4];
#pragma unroll
                        for (int u = 0; u < 4; u++) Rf[u] = ok[u] ? R::load(H + f[u]) : FF;
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            if (!ok[u]) continue;
                            p_edges++;
                            RowT le = R::le(Rf[u], L);
                            if (!(blocking && le == (RowT)~(RowT)0)) found |= le & inf;
                        }
                        if (!ok[3]) break;  // activation-sorted: past the gate (or the row end)
                    }
                    if (found && vpx) {
                        vp_set_bits<RowT>(vpx, blockIdx.y, wc, n - lo, found);
                    } else if (found) {
                        RowT nr = (Rn & ~found) | (found & R::splat(l + 1));
                        *(H + n) = nr;
                        enq = true;
                        id = collect && R::eq(nr, FF) == 0;
                        p_cells += R::ones(found);
                    }
                }
            }
            frontier_push(w, enq, s, n, nxt);
            cand_push(g, w, id, s, n, l + 1);
        }
    }
    p_nodes = warp_sum(p_nodes);
    p_edges = warp_sum(p_edges);
    p_cells = warp_sum(p_cells);
    if (lane == 0 && (p_nodes | p_edges)) {
        atomicAdd(&w.prof[P_PULLNODES], (unsigned long long)p_nodes);
        atomicAdd(&w.prof[P_PULLEDGES], (unsigned long long)p_edges);
        atomicAdd(&w.prof[P_NEWCELLS], (unsigned long long)p_cells);
    }
}

// ====================================================================== joint traversal
// Joint multi-query expansion (iBFS-style sharing of the adjacency reads
// across the queries of a batch).  H is node-major: the rows of all SP slots of node n are
// contiguous, so a warp reads them with one 16-byte load per lane (lane c owns slots
// [c*16/RB, (c+1)*16/RB)).  The frontier is the union over slots (bit-packed flags dedup
// it); each frontier node and each of its due edges is visited ONCE per level for the
// whole batch, and every slot applies exactly its own Alg. 1 rule through byte masks: new
// columns (h == l) relax edges with a <= l, old columns (h < l) edges with a == l, CF-blocked
// slots and slots outside the run nothing.  Relaxation, first-writer and completion logic
// per slot is the same atomicAnd as in k_expand, on the 32-bit word holding the slot rows.
constexpr uint32_t JHEAVY = 512, JCHUNK = 512;

template <int RB> __device__ __forceinline__ uint32_t slot_bytes(int h) {
    return RB == 4 ? 0xFFFFFFFFu : (h ? 0xFFFF0000u : 0x0000FFFFu);
}
template <int RB> __device__ __forceinline__ uint32_t full_slots(uint32_t m) {  // slots whose bytes are all set
    if (RB == 4) return m == 0xFFFFFFFFu ? 0xFFFFFFFFu : 0u;
    return ((m & 0xFFFFu) == 0xFFFFu ? 0xFFFFu : 0u) | ((m >> 16) == 0xFFFFu ? 0xFFFF0000u : 0u);
}
template <int RB> __device__ __forceinline__ uint32_t any_slots(uint32_t m) {  // slots with any byte set
    if (RB == 4) return m ? 0xFFFFFFFFu : 0u;
    return ((m & 0xFFFFu) ? 0xFFFFu : 0u) | ((m & 0xFFFF0000u) ? 0xFFFF0000u : 0u);
}
__device__ __forceinline__ uint32_t u4w(const uint4 &v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }

// push node n to the next union frontier (bit-packed dedup); convergent
__device__ __forceinline__ void jq_push(const WsDev &w, bool want, uint32_t n, uint32_t nxt) {
    bool app = false;
    if (want) {
        uint32_t bit = 1u << (n & 31);
        app = !(atomicOr(w.JBM(nxt) + (n >> 5), bit) & bit);
    }
    uint32_t pos = warp_append(app, 0, &w.ctr[C_JQN0 + nxt], 0);
    if (app) w.JQ(nxt)[pos] = n;
}

template <class RowT, bool HEAVYP>
__global__ void __launch_bounds__(256) k_jexpand(GraphDev g, WsDev w, int ph, uint32_t l) {
    constexpr int RB = sizeof(RowT), SPW = 4 / RB, PER = 16 / RB;
    __shared__ uint32_t s_cnt[256];
    __shared__ uint32_t s_info[256];
    __shared__ uint8_t s_ne[256];
    const uint32_t SP = w.SP, lane = lane_id();
    for (uint32_t i = threadIdx.x; i < SP; i += blockDim.x) {
        s_cnt[i] = 0;
        s_ne[i] = 0;
        uint32_t info = 0;
        if (i < w.nslots) {
            const SlotState &st = w.st[i];
            info = st.in_phase | st.blocking << 1 | st.collect << 2 | st.T[ph] << 8;
        }
        s_info[i] = info;
    }
    __syncthreads();
    // per-lane word masks of its slots: used columns of slots in the run, blocking, collect
    uint32_t usedw[4], blkw[4], colw[4];
    const bool lv = lane * 16 < SP * RB;
#pragma unroll
    for (int wi = 0; wi < 4; wi++) {
        usedw[wi] = blkw[wi] = colw[wi] = 0;
#pragma unroll
        for (int h = 0; h < SPW; h++) {
            uint32_t sl = lane * PER + wi * SPW + h;
            uint32_t info = lv && sl < SP ? s_info[sl] : 0;
            if (!(info & 1)) continue;
            uint32_t T = min(info >> 8, (uint32_t)RB);
            uint32_t um = T >= 4 ? 0xFFFFFFFFu : ((1u << (8 * T)) - 1);
            usedw[wi] |= um << (8 * RB * h);
            if (info & 2) blkw[wi] |= slot_bytes<RB>(h);
            if (info & 4) colw[wi] |= slot_bytes<RB>(h);
        }
    }
    const uint32_t L = l * 0x01010101u, L1 = (l + 1) * 0x01010101u;
    const uint32_t cur = l & 1, nxt = cur ^ 1;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t nitems = HEAVYP ? min(w.ctr[C_JHEAVY], w.heavy_cap) : w.ctr[C_JQCUR];
    uint8_t *Hb = w.H[ph];
    const size_t rowb = (size_t)SP * RB;
    uint32_t p_items = 0, p_edges = 0, p_cells = 0, p_enq = 0;
    for (uint32_t it = gw; it < nitems; it += nw) {
        uint32_t f, lo = 0, hi = 0, eqlo = 0;
        if (HEAVYP) {
            uint4 hh = w.heavy[it];
            f = hh.x; lo = hh.y; hi = hh.z; eqlo = hh.w;
        } else {
            f = w.JQ(cur)[it];
            if (lane == 0) w.JBM(cur)[f >> 5] = 0;  // every flag of this word is a node of this queue
        }
        const uint4 Rf = lv ? __ldcg((const uint4 *)(Hb + f * rowb) + lane) : make_uint4(0, 0, 0, 0);
        uint32_t newc[4], oldc[4];
#pragma unroll
        for (int wi = 0; wi < 4; wi++) {
            uint32_t R = u4w(Rf, wi);
            uint32_t blocked = full_slots<RB>(__vcmpleu4(R, L)) & blkw[wi];  // CF per slot (R10)
            newc[wi] = __vcmpeq4(R, L) & usedw[wi] & ~blocked;
            oldc[wi] = __vcmpltu4(R, L) & usedw[wi] & ~blocked;
        }
        const bool any_new = __any_sync(FULLMASK, (newc[0] | newc[1] | newc[2] | newc[3]) != 0);
        const bool any_old = __any_sync(FULLMASK, (oldc[0] | oldc[1] | oldc[2] | oldc[3]) != 0);
        if (!any_new && !any_old) continue;
        if (!HEAVYP) {
            p_items++;
            const uint4 d = __ldg(g.desc + f);
            const uint32_t rb = d.x, re = d.x + d.y;
            gate_range(g, d, l, hi, eqlo);
            lo = any_new ? rb : eqlo;
            // per-slot relaxation counts and retention (Alg. 1 lines 9-11)
            bool retain_any = false;
#pragma unroll
            for (int wi = 0; wi < 4; wi++) {
#pragma unroll
                for (int h = 0; h < SPW; h++) {
                    uint32_t sb = slot_bytes<RB>(h);
                    uint32_t nc = newc[wi] & sb, oc = oldc[wi] & sb;
                    if (!(nc | oc)) continue;
                    uint32_t sl = lane * PER + wi * SPW + h;
                    uint32_t cnt = (hi - rb) * (__popc(nc) >> 3) + (hi - eqlo) * (__popc(oc) >> 3);
                    if (cnt) atomicAdd(&s_cnt[sl], cnt);
                    if (hi < re) { s_ne[sl] = 1; retain_any = true; }
                }
            }
            const bool ret = __any_sync(FULLMASK, retain_any);
            jq_push(w, ret && lane == 0, f, nxt);
            p_enq += ret && lane == 0;
            if (hi - lo > JHEAVY) {  // hub rows: chunks for the heavy pass
                if (lane == 0) {
                    uint32_t nch = (hi - lo + JCHUNK - 1) / JCHUNK;
                    uint32_t p = atomicAdd(&w.ctr[C_JHEAVY], nch);
                    if (p + nch <= w.heavy_cap) {
                        for (uint32_t c = 0; c < nch; c++)
                            w.heavy[p + c] = make_uint4(f, lo + c * JCHUNK, min(lo + (c + 1) * JCHUNK, hi), eqlo);
                    } else {
                        atomicOr(&w.st[0].err, (uint32_t)E_HEAVY);
                    }
                }
                p_edges += hi - lo;
                continue;
            }
            p_edges += hi - lo;
        }
        // edges: 4 per iteration, all 32 lanes on each edge (lane = slot group)
        for (uint32_t e0 = lo; e0 < hi; e0 += 4) {
            uint32_t nn[4];
            uint4 Rn[4];
#pragma unroll
            for (int u = 0; u < 4; u++) nn[u] = e0 + u < hi ? __ldg(g.col + e0 + u) : 0;
#pragma unroll
            for (int u = 0; u < 4; u++)
                Rn[u] = (lv && e0 + u < hi) ? __ldcg((const uint4 *)(Hb + nn[u] * rowb) + lane) : make_uint4(0, 0, 0, 0);
            bool firstq[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const bool isold = e0 + u >= eqlo;
                bool lane_first = false;
                uint32_t cmpk = 0;  // bit k: slot k of this lane completed its row (identification)
                if (e0 + u < hi) {
#pragma unroll
                    for (int wi = 0; wi < 4; wi++) {
                        uint32_t need = (newc[wi] | (isold ? oldc[wi] : 0u)) & __vcmpeq4(u4w(Rn[u], wi), 0xFFFFFFFFu);
                        if (!need) continue;
                        uint32_t andm = ~need | (need & L1);
                        uint32_t *addr = (uint32_t *)(Hb + nn[u] * rowb) + lane * 4 + wi;
                        uint32_t old = atomicAnd(addr, andm);
                        uint32_t changed = need & __vcmpeq4(old, 0xFFFFFFFFu);
                        if (!changed) continue;
                        p_cells += __popc(changed) >> 3;
                        uint32_t chs = any_slots<RB>(changed);
                        uint32_t fst = chs & ~any_slots<RB>(__vcmpeq4(old, L1));
                        uint32_t cmp = chs & ~any_slots<RB>(__vcmpeq4(old & andm, 0xFFFFFFFFu)) & colw[wi];
#pragma unroll
                        for (int h = 0; h < SPW; h++) {
                            uint32_t sb = slot_bytes<RB>(h);
                            if (fst & sb) { s_ne[lane * PER + wi * SPW + h] = 1; lane_first = true; }
                            if (cmp & sb) cmpk |= 1u << (wi * SPW + h);
                        }
                    }
                }
                firstq[u] = __any_sync(FULLMASK, lane_first);
                if (__any_sync(FULLMASK, cmpk != 0)) {
#pragma unroll
                    for (int k = 0; k < PER; k++) cand_push(g, w, (cmpk >> k) & 1, lane * PER + k, nn[u], l + 1);
                }
            }
            // union-frontier pushes for the (up to) 4 relaxed targets: lane u pushes edge u
            bool want = false;
            uint32_t tn = 0;
#pragma unroll
            for (int u = 0; u < 4; u++)
                if (lane == (uint32_t)u) { want = firstq[u]; tn = nn[u]; }
            jq_push(w, want, tn, nxt);
            p_enq += want;
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < SP && i < w.nslots; i += blockDim.x) {
        if (s_ne[i]) w.st[i].nq[nxt] = 1;  // Phi_{l+1}(slot) is not empty
        if (s_cnt[i]) atomicAdd(&w.st[i].relax[ph], (unsigned long long)s_cnt[i]);
    }
    p_items = warp_sum(p_items);
    p_edges = warp_sum(p_edges);
    p_cells = warp_sum(p_cells);
    p_enq = warp_sum(p_enq);
    if (lane == 0 && (p_items | p_edges | p_cells)) {
        atomicAdd(&w.prof[P_ITEMS], (unsigned long long)p_items);
        atomicAdd(&w.prof[P_EDGES], (unsigned long long)p_edges);
        atomicAdd(&w.prof[P_NEWCELLS], (unsigned long long)p_cells);
        atomicAdd(&w.prof[P_ENQ], (unsigned long long)p_enq);
    }
}

// clear the flags of the last (unconsumed) union frontier of a run
__global__ void k_jclear(WsDev w, uint32_t b) {
    uint32_t n = w.ctr[C_JQN0 + b];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        w.JBM(b)[w.JQ(b)[i] >> 5] = 0;
}

// ====================================================================== candidates
__device__ void cta_sort_u64(uint64_t *keys, uint32_t n, uint64_t *smem, uint32_t smem_cap) {
    if (n < 2) return;
    if (next_pow2(n) <= smem_cap) {
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) smem[i] = keys[i];
        __syncthreads();
        cta_bitonic_sort(smem, n);
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) keys[i] = smem[i];
        __syncthreads();
    } else {
        cta_bitonic_sort(keys, n);  // global buffer has capacity next_pow2(n) (capc is a power of 2)
    }
}

// Segments of the candidate-key sort: slot s's keys CK(s)[0, ncand) (empty for slots that
// are inactive or failed).
// Offsets are relative to the first slot of s's sort group (G slots: int-sized item counts).
__global__ void k_cand_segments(WsDev w, int *begin, int *end, uint32_t G) {
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= w.nslots) return;
    const SlotState &st = w.st[s];
    begin[s] = (int)((size_t)(s % G) * w.capc);
    end[s] = begin[s] + ((st.active && !st.err) ? (int)min(st.ncand, w.capc) : 0);
}

// Candidate CGs: all CGs identified by the terminating level, ties kept (R13), ordered
// by (S^c, v); beam_mode 1 truncates to the first w.  `sorted` holds every slot's keys
// already sorted (segmented radix sort of CK, keys (S^c << 32 | caller id)); they are copied
// back to CK(s) while the candidate records are built.
__global__ void k_cand_sort(GraphDev g, WsDev w, const uint64_t *sorted) {
    uint32_t s = blockIdx.x;
    SlotState &st = w.st[s];
    if (!st.active || st.err) {
        if (threadIdx.x == 0) st.ncand_kept = st.n_extract = 0;
        return;
    }
    uint32_t n = min(st.ncand, w.capc);
    const uint64_t *src = sorted + (size_t)s * w.capc;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) w.CK(s)[i] = src[i];
    // beam_mode 1 with the tie-break (R29) truncates by (S^c, W(CG), v) after recovery
    const bool beam_tie = st.beam_mode == 1 && st.tie_break;
    uint32_t kept = st.beam_mode == 1 && !beam_tie ? min(n, st.w) : n;
    uint32_t nex = st.T[1] == 0 && !st.tie_break ? min(kept, st.k) : kept;
    for (uint32_t i = threadIdx.x; i < nex; i += blockDim.x) {
        uint64_t key = src[i];
        Cand c;
        memset(&c, 0, sizeof(c));
        c.ext = (uint32_t)key;
        c.v = g.perm[c.ext];
        c.sc = (uint32_t)(key >> 32);
        c.sr = (double)c.sc;
        c.ptc = 1;
        w.CD(s)[i] = c;
        w.CST(s)[i] = 0;
    }
    if (threadIdx.x == 0) {
        st.ncand_kept = kept;
        st.n_extract = nex;
    }
}

__global__ void k_scan_cands(WsDev w) {
    __shared__ uint32_t sc[MAX_SLOTS];
    uint32_t s = threadIdx.x;
    uint32_t v = s < w.nslots ? w.st[s].n_extract : 0;
    sc[s] = v;
    __syncthreads();
    for (uint32_t o = 1; o < MAX_SLOTS; o <<= 1) {
        uint32_t t = s >= o ? sc[s - o] : 0;
        __syncthreads();
        sc[s] += t;
        __syncthreads();
    }
    if (s < w.nslots) w.coffs[s] = sc[s] - v;
    if (s == 0) {
        w.coffs[w.nslots] = sc[MAX_SLOTS - 1];
        w.ctr[C_NCAND_TOTAL] = sc[MAX_SLOTS - 1];
        w.ctr[C_RECQ] = 0;
        w.ctr[C_NOVF] = 0;
        w.ctr[C_NOVF2] = 0;
    }
}

// ====================================================================== recovery (Alg. 2)
// Recovery code is written for a "group" of threads that cooperates on one candidate: a
// single warp (fast tier, no block barriers) or a whole CTA (bigger tiers).
struct GroupWarp {
    __device__ __forceinline__ uint32_t rank() const { return lane_id(); }
    __device__ __forceinline__ uint32_t size() const { return 32; }
    __device__ __forceinline__ uint32_t warp() const { return 0; }
    __device__ __forceinline__ uint32_t nwarps() const { return 1; }
    __device__ __forceinline__ void sync() const { __syncwarp(); }
};
struct GroupCTA {
    __device__ __forceinline__ uint32_t rank() const { return threadIdx.x; }
    __device__ __forceinline__ uint32_t size() const { return blockDim.x; }
    __device__ __forceinline__ uint32_t warp() const { return threadIdx.x >> 5; }
    __device__ __forceinline__ uint32_t nwarps() const { return blockDim.x >> 5; }
    __device__ __forceinline__ void sync() const { __syncthreads(); }
};

// Hash set of node ids that records its insertions (items = insertion order, slots = where
// they live), so clearing and enumerating cost O(inserted), not O(capacity).
struct HSet {
    uint32_t *keys, *items, *slots;
    uint32_t cap, items_cap;  // cap: power of two
    uint32_t *count;          // shared/global counter
    // returns the insertion index (>= 0), -1 if k was present, -2 on overflow
    __device__ __forceinline__ int insert(uint32_t k, uint32_t *ovf) const {
        uint32_t h = HashSet::hash(k) & (cap - 1);
        for (uint32_t i = 0; i < cap; i++) {
            uint32_t sl = (h + i) & (cap - 1);
            uint32_t prev = atomicCAS(&keys[sl], EMPTY, k);
            if (prev == EMPTY) {
                uint32_t idx = atomicAdd(count, 1u);
                if (idx < items_cap) { items[idx] = k; slots[idx] = sl; return (int)idx; }
                *ovf = 1;
                return -2;
            }
            if (prev == k) return -1;
        }
        *ovf = 1;
        return -2;
    }
    __device__ __forceinline__ int find(uint32_t k) const {
        uint32_t h = HashSet::hash(k) & (cap - 1);
        for (uint32_t i = 0; i < cap; i++) {
            uint32_t sl = (h + i) & (cap - 1);
            uint32_t v = keys[sl];
            if (v == k) return (int)sl;
            if (v == EMPTY) return -1;
        }
        return -1;
    }
    template <class G> __device__ __forceinline__ void clear_inserted(const G &G_, bool full) const {
        uint32_t n = min(*count, items_cap);
        if (full) for (uint32_t i = G_.rank(); i < cap; i += G_.size()) keys[i] = EMPTY;
        else for (uint32_t i = G_.rank(); i < n; i += G_.size()) keys[slots[i]] = EMPTY;
    }
};

struct ExBuf {
    HSet hu, hk;          // union of nodes; per-keyword visited set whose items are the BFS queue
    uint8_t *qh;          // hitting level of each queue item (parallel to hk.items)
    uint32_t *edges, *uf;
    uint8_t *flag;
    uint32_t cap_e;
};
struct ExShared {
    uint32_t nu, nk, nedges, ovf;
    uint32_t cnt, off, mnr, mxr, nx, xvc;
    uint32_t dirty;  // tables may hold unrecorded entries (after an overflow): full clear needed
};

// ---- memoised recovery DAG.  The Alg. 2 predicate (Lemma recover P:553 + R16) does not
// depend on the candidate, so the predecessor list of (slot, phase, column j, node q) is
// computed once and shared by every candidate of the query through a per-slot map with a
// claim/publish protocol (a claimer never waits, so spinning readers always progress).
constexpr uint32_t MAPCAP = 8192;
constexpr unsigned long long NOT_READY = ~0ull;

// Map entry (16 B): {key, -, (cnt, off) as one 64-bit word}; one 16-byte load finds a
// published list.  List entries are 3 words: (n, caller edge id, h_n).  Called by a warp.
template <class RowT>
__device__ void dag_list(const GraphDev &g, const WsDev &w, uint32_t s, int ph, int j, const HV<RowT> H, bool blocking,
                         uint32_t q, uint32_t hq, uint32_t *off_out, uint32_t *cnt_out) {
    typedef Row<RowT> R;
    const uint32_t lane = lane_id();
    uint4 *tab = w.mtab + ((size_t)s * 16 + ph * 8 + j) * MAPCAP;
    int state = 0;  // 0 full (compute, no cache), 1 claimed (compute + publish), 2 found
    uint32_t slot = 0;
    unsigned long long v = NOT_READY;
    if (lane == 0) {
        uint32_t h = HashSet::hash(q) & (MAPCAP - 1);
        for (uint32_t i = 0; i < 64; i++) {  // bounded probe: a full neighbourhood just disables caching
            uint32_t sl = (h + i) & (MAPCAP - 1);
            uint4 e = __ldcg(tab + sl);
            if (e.x == q) { state = 2; slot = sl; v = (unsigned long long)e.w << 32 | e.z; break; }
            if (e.x == EMPTY) {
                uint32_t prev = atomicCAS(&tab[sl].x, EMPTY, q);
                if (prev == EMPTY) { state = 1; slot = sl; break; }
                if (prev == q) { state = 2; slot = sl; break; }
            }
        }
        if (state == 2 && v == NOT_READY) {
#if REC_STATS
            const long long t0 = clock64();
#endif
            volatile unsigned long long *vv = (volatile unsigned long long *)&tab[slot].z;
            while ((v = *vv) == NOT_READY) __nanosleep(32);
#if REC_STATS
            atomicAdd(&w.prof[P_R_WAITS], 1ull);
            atomicAdd(&w.prof[P_R_WCYC], (unsigned long long)(clock64() - t0));
#endif
        }
    }
    state = __shfl_sync(FULLMASK, state, 0);
    if (state == 2) {  // list reads below depend on (off, cnt) and go through L2 (__ldcg)
        v = __shfl_sync(FULLMASK, v, 0);
        *off_out = (uint32_t)(v >> 32);
        *cnt_out = (uint32_t)v;
        return;
    }
    slot = __shfl_sync(FULLMASK, slot, 0);
#if REC_STATS
    const long long tb0 = clock64();
#endif
    const uint4 d = __ldg(g.idesc + q);  // in-rows are activation-sorted: gate a <= hq - 1
    const uint32_t rb = d.x;
    uint32_t hi, eqlo;
    gate_range_in(g, d, hq - 1, hi, eqlo);
    uint32_t off = 0;
    if (lane == 0) {
        unsigned long long p = atomicAdd(w.arena_used, 3ull * (hi - rb));
        if (p + 3ull * (hi - rb) > w.arena_cap) { atomicOr(&w.st[s].err, (uint32_t)E_ARENA); off = EMPTY; }
        else off = (uint32_t)p;
    }
    off = __shfl_sync(FULLMASK, off, 0);
    uint32_t cnt = 0;
    if (off != EMPTY) {
        for (uint32_t k0 = rb; k0 < hi; k0 += 128) {
            uint32_t n[4], a[4], hn[4];
            RowT Rn[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                uint32_t k = k0 + u * 32 + lane;
                n[u] = k < hi ? __ldg(g.isrc + k) : 0;
                a[u] = k < hi ? __ldg(g.iact + k) : 0xFF;
            }
#pragma unroll
            for (int u = 0; u < 4; u++) Rn[u] = (k0 + u * 32 + lane < hi) ? R::load(H + n[u]) : R::splat(0xFF);
#pragma unroll
            for (int u = 0; u < 4; u++) {
                uint32_t k = k0 + u * 32 + lane;
                hn[u] = R::byte(Rn[u], j);
                bool ok = false;
                if (k < hi && hn[u] != 0xFF) {
                    uint32_t Lr = max(hn[u], a[u]);
                    if (Lr + 1 == hq) {
                        uint32_t blk = 0xFF;
                        if (blocking && R::eq(Rn[u], R::splat(0xFF)) == 0) blk = R::maxb(Rn[u]);
                        ok = Lr < blk;
                    }
                }
                uint32_t m = __ballot_sync(FULLMASK, ok);
                if (ok) {
                    uint32_t p = off + 3 * (cnt + __popc(m & lanemask_lt()));
                    w.arena[p] = n[u];
                    w.arena[p + 1] = __ldg(g.ieid + k);
                    w.arena[p + 2] = hn[u];
                }
                cnt += __popc(m);
            }
        }
    }
    if (state == 1 && lane == 0) {
        __threadfence();
        atomicExch((unsigned long long *)&tab[slot].z, off == EMPTY ? 0ull : ((unsigned long long)off << 32 | cnt));
    }
#if REC_STATS
    if (lane == 0) {
        atomicAdd(&w.prof[P_R_BUILDS], 1ull);
        atomicAdd(&w.prof[P_R_BEDGES], (unsigned long long)(hi - rb));
        atomicMax(&w.prof[P_R_BMAX], (unsigned long long)(hi - rb));
        atomicAdd(&w.prof[P_R_BCYC], (unsigned long long)(clock64() - tb0));
    }
#endif
    *off_out = off == EMPTY ? 0 : off;
    *cnt_out = off == EMPTY ? 0 : cnt;
}

// Reverse BFS for keyword column j (Alg. 2 lines 4-10): edge (n -> q) is recovered iff it
// is in q's DAG list; n is continued from iff h_nj != 0 (line 10) and unvisited (R17).
// hk.items (the queue) and qh hold the sources and their levels on entry.
template <class G, class RowT>
__device__ void bfs_column(const G &G_, const GraphDev &g, const WsDev &w, uint32_t s, int ph, int j, const HV<RowT> H,
                           bool blocking, const ExBuf &b, ExShared &sh) {
    const uint32_t lane = lane_id(), warp = G_.warp(), nw = G_.nwarps();
    uint32_t head = 0, tail = min(sh.nk, b.hk.items_cap);
    while (head < tail) {
        for (uint32_t it = head + warp; it < tail; it += nw) {
            uint32_t q = b.hk.items[it];
            uint32_t hq = b.qh[it];
            if (hq == 0 || hq == 0xFF) continue;
#if REC_STATS
            if (lane == 0) atomicAdd(&w.prof[P_R_ITEMS], 1ull);
#endif
            uint32_t off, cnt;
            dag_list<RowT>(g, w, s, ph, j, H, blocking, q, hq, &off, &cnt);
            for (uint32_t t = lane; t < cnt; t += 32) {
                uint32_t n = __ldcg(w.arena + off + 3 * t), eid = __ldcg(w.arena + off + 3 * t + 1);
                uint32_t hn = __ldcg(w.arena + off + 3 * t + 2);
                uint32_t pos = atomicAdd(&sh.nedges, 1u);
                if (pos < b.cap_e) b.edges[pos] = eid; else sh.ovf = 1;
                b.hu.insert(n, &sh.ovf);
                if (hn != 0) {
                    int idx = b.hk.insert(n, &sh.ovf);
                    if (idx >= 0) b.qh[idx] = (uint8_t)hn;
                }
            }
        }
        G_.sync();
        head = tail;
        tail = min(sh.nk, b.hk.items_cap);
        bool stop = sh.ovf;
        G_.sync();
        if (stop) break;
    }
}

// Tier-0 recovery work distribution: every warp starts on item `first` (< stride); with
// REC_DYNAMIC the next items come from a shared counter (ctr[C_RECQ], zeroed before the
// launch) in index order, so a warp stuck on a long predecessor-list build does not hold
// back a fixed share of the items; otherwise the static cyclic stride.
#ifndef REC_DYNAMIC
#define REC_DYNAMIC 0
#endif
__device__ __forceinline__ uint32_t rec_next(const WsDev &w, uint32_t item, uint32_t stride) {
#if REC_DYNAMIC
    uint32_t nx = 0;
    if (lane_id() == 0) nx = stride + atomicAdd(&w.ctr[C_RECQ], 1u);
    return __shfl_sync(FULLMASK, nx, 0);
#else
    return item + stride;
#endif
}

__device__ __forceinline__ uint32_t arena_alloc(const WsDev &w, uint32_t words, uint32_t s) {
    unsigned long long p = atomicAdd(w.arena_used, (unsigned long long)words);
    if (p + words > w.arena_cap) {
        atomicOr(&w.st[s].err, (uint32_t)E_ARENA);
        return EMPTY;
    }
    return (uint32_t)p;
}

template <class G> __device__ __forceinline__ void ex_reset(const G &G_, const ExBuf &b, ExShared &sh) {
    bool full = sh.dirty;
    b.hu.clear_inserted(G_, full);
    b.hk.clear_inserted(G_, full);
    G_.sync();
    if (G_.rank() == 0) { sh.nu = 0; sh.nk = 0; sh.nedges = 0; sh.ovf = 0; sh.dirty = 0; }
    G_.sync();
}
template <class G> __device__ __forceinline__ void ex_reset_hk(const G &G_, const ExBuf &b, ExShared &sh) {
    b.hk.clear_inserted(G_, sh.dirty != 0);
    G_.sync();
    if (G_.rank() == 0) sh.nk = 0;
    G_.sync();
}
template <class G> __device__ __forceinline__ void ex_init(const G &G_, const ExBuf &b, ExShared &sh) {
    if (G_.rank() == 0) sh.dirty = 1;
    G_.sync();
    ex_reset(G_, b, sh);
}
// Global-scratch tier: its V-sized tables are EMPTY on entry (filled with 0xFF when the
// workspace is allocated, and every use leaves them clean: ex_reset clears the inserted
// entries, or everything after an overflow), so no O(V) clear per launch.
template <class G> __device__ __forceinline__ void ex_init_clean(const G &G_, ExShared &sh) {
    if (G_.rank() == 0) { sh.nu = 0; sh.nk = 0; sh.nedges = 0; sh.ovf = 0; sh.dirty = 0; }
    G_.sync();
}

// CG of candidate (s, c): union over central keywords of the recovered SP(c_j, v~).
// Writes nodes, edge ids and V_C (nodes holding a central keyword) to the arena.
template <class G, class RowC> __device__ void extract_cg(const G &G_, const GraphDev &g, const WsDev &w, uint32_t s,
                                                          uint32_t c, const ExBuf &b, ExShared &sh, bool *overflow) {
    typedef Row<RowC> R;
    const SlotState &st = w.st[s];
    Cand &cd = w.CD(s)[c];
    const HV<RowC> H = w.Hs<RowC>(0, s);
    const uint32_t T = st.T[0];
    const uint32_t v = cd.v;
    if (G_.rank() == 0) b.hu.insert(v, &sh.ovf);
    const RowC Rv = R::load(H + v);
    for (uint32_t j = 0; j < T; j++) {
        if (G_.rank() == 0) {
            int idx = b.hk.insert(v, &sh.ovf);
            if (idx >= 0) b.qh[idx] = (uint8_t)R::byte(Rv, j);
        }
        G_.sync();
        bfs_column(G_, g, w, s, 0, j, H, true, b, sh);
        if (sh.ovf) break;
        ex_reset_hk(G_, b, sh);
    }
    G_.sync();
    if (sh.ovf) { *overflow = true; return; }
    *overflow = false;
    const uint32_t nn = min(sh.nu, b.hu.items_cap), ne = min(sh.nedges, b.cap_e);
    RowC used = used_mask<RowC>(T);
    if (G_.rank() == 0) sh.cnt = 0;
    G_.sync();
    for (uint32_t i = G_.rank(); i < nn; i += G_.size())
        if (R::eq(R::load(H + b.hu.items[i]), 0) & used) atomicAdd(&sh.cnt, 1u);
    G_.sync();
    const uint32_t nvc = sh.cnt;
    G_.sync();
    if (G_.rank() == 0) { sh.off = arena_alloc(w, nn + ne + nvc, s); sh.cnt = 0; }
    G_.sync();
    const uint32_t off = sh.off;
    if (off != EMPTY) {
        for (uint32_t i = G_.rank(); i < nn; i += G_.size()) {
            uint32_t x = b.hu.items[i];
            w.arena[off + i] = x;
            if (R::eq(R::load(H + x), 0) & used) w.arena[off + nn + ne + atomicAdd(&sh.cnt, 1u)] = x;
        }
        for (uint32_t i = G_.rank(); i < ne; i += G_.size()) w.arena[off + nn + i] = b.edges[i];
    }
    G_.sync();
    if (G_.rank() == 0 && off != EMPTY) {
        cd.nodes_off = off; cd.n_nodes = nn;
        cd.edges_off = off + nn; cd.n_edges = ne;
        cd.vc_off = off + nn + ne; cd.n_vc = nvc;
    }
}

// Tiers: 0 = one warp per candidate with 7 KB of shared memory (4 warps per CTA);
// 1 = one CTA (256 threads) per candidate with 58 KB; 2 = global scratch sized by V.  A
// candidate that overflows a tier is re-run by the next one, so recovery is exact at any size.
template <int TIER> struct Tier;
#ifndef T0_FE
#define T0_FE 256
#endif
#ifndef T0_GROUPS
#define T0_GROUPS 6
#endif
template <> struct Tier<0> { static constexpr uint32_t FU = 256, FUI = 128, FK = 256, FKI = 128, FE = T0_FE, GROUPS = T0_GROUPS; };
template <> struct Tier<1> { static constexpr uint32_t FU = 2048, FUI = 1024, FK = 2048, FKI = 1024, FE = 4096, GROUPS = 1; };
template <int TIER> constexpr size_t smem_group() {
    return ((size_t)(Tier<TIER>::FU + 2 * Tier<TIER>::FUI + Tier<TIER>::FK + 2 * Tier<TIER>::FKI + Tier<TIER>::FE +
                     Tier<TIER>::FU) * 4 + Tier<TIER>::FU + Tier<TIER>::FKI + 15) & ~(size_t)15;
}
template <int TIER> constexpr size_t smem_ex() { return smem_group<TIER>() * Tier<TIER>::GROUPS; }
template <int TIER> constexpr uint32_t tier_threads() { return TIER == 0 ? 32 * Tier<0>::GROUPS : 256; }

template <int TIER> __device__ __forceinline__ ExBuf smem_buf(uint8_t *sm, ExShared &sh) {
    typedef Tier<TIER> C;
    uint32_t *p = (uint32_t *)sm;
    ExBuf b;
    b.hu = HSet{p, p + C::FU, p + C::FU + C::FUI, C::FU, C::FUI, &sh.nu};
    p += C::FU + 2 * C::FUI;
    b.hk = HSet{p, p + C::FK, p + C::FK + C::FKI, C::FK, C::FKI, &sh.nk};
    p += C::FK + 2 * C::FKI;
    b.edges = p; b.cap_e = C::FE;
    p += C::FE;
    b.uf = p;
    b.flag = (uint8_t *)(p + C::FU);
    b.qh = b.flag + C::FU;
    return b;
}

__device__ __forceinline__ ExBuf big_buf(const WsDev &w, uint32_t cta, ExShared &sh) {
    // global scratch for the last tier; capacities scale with V
    uint32_t *p = w.big + w.big_words * cta;
    const uint32_t cu = next_pow2(2 * w.V + 2), ni = w.V + 1;
    ExBuf b;
    b.hu = HSet{p, p + cu, p + cu + ni, cu, ni, &sh.nu};
    p += cu + 2 * ni;
    b.hk = HSet{p, p + cu, p + cu + ni, cu, ni, &sh.nk};
    p += cu + 2 * ni;
    b.uf = p;
    p += cu;
    b.flag = (uint8_t *)p;
    p += cu / 4 + 4;
    b.qh = (uint8_t *)p;
    p += ni / 4 + 4;
    b.edges = p;
    unsigned long long rem = w.big_words - (unsigned long long)(p - (w.big + w.big_words * cta));
    b.cap_e = (uint32_t)(rem < 0xFFFFFFFFull ? rem : 0xFFFFFFFFull);
    return b;
}

// overflow hand-off to the next tier
__device__ __forceinline__ void push_overflow(const WsDev &w, int tier, uint2 sc) {
    uint32_t *ctr = &w.ctr[tier == 0 ? C_NOVF : C_NOVF2];
    uint2 *lst = tier == 0 ? w.ovf : w.ovf2;
    uint32_t p = atomicAdd(ctr, 1u);
    if (p < w.ovf_cap) lst[p] = sc; else atomicOr(&w.st[sc.x].err, (uint32_t)E_EXTRACT);
}

// Tier 0 takes the candidates from the flattened (slot, candidate) range (one warp each);
// tier 1 and tier 2 take the overflow list of the previous tier.
template <class RowC, int TIER> __global__ void __launch_bounds__(tier_threads<TIER>()) k_extract_cg(GraphDev g, WsDev w) {
    extern __shared__ __align__(16) uint8_t smx[];
    __shared__ ExShared shs[Tier<TIER>::GROUPS];
    const uint32_t total = TIER == 0 ? w.coffs[w.nslots] : min(w.ctr[C_NOVF], w.ovf_cap);
    const uint32_t gi = TIER == 0 ? threadIdx.x >> 5 : 0;
    ExShared &sh = shs[gi];
    ExBuf b = smem_buf<TIER>(smx + smem_group<TIER>() * gi, sh);
    const uint32_t first = blockIdx.x * Tier<TIER>::GROUPS + gi, stride = gridDim.x * Tier<TIER>::GROUPS;
    if (TIER == 0) {
        GroupWarp G_;
        if (first >= total) return;
        ex_init(G_, b, sh);
#if REC_STATS
        unsigned long long wsum = 0;
#endif
        // cyclic distribution: concurrent warps share queries (their H arrays and memo lists stay
        // hot in L2), which measured faster than spreading warps over queries
        for (uint32_t item = first; item < total; item = rec_next(w, item, stride)) {
            uint32_t s = find_slot(w.coffs, w.nslots, item), c = item - w.coffs[s];
            bool ovf = false;
#if REC_STATS
            const long long tc0 = clock64();
#endif
            extract_cg<GroupWarp, RowC>(G_, g, w, s, c, b, sh, &ovf);
#if REC_STATS
            if (G_.rank() == 0) {
                const unsigned long long dt = clock64() - tc0;
                atomicAdd(&w.prof[P_R_CANDS], 1ull);
                atomicAdd(&w.prof[P_R_CANDCYC], dt);
                atomicMax(&w.prof[P_R_CANDMAX], dt);
                const int bk = dt < 16384 ? 0 : dt < 65536 ? 1 : dt < 262144 ? 2 : dt < 1048576 ? 3 : dt < 4194304 ? 4 : 5;
                atomicAdd(&w.prof[P_R_H0 + bk], 1ull);
                wsum += dt;
            }
#endif
            if (ovf && G_.rank() == 0) { sh.dirty = 1; push_overflow(w, 0, make_uint2(s, c)); }
            G_.sync();
            ex_reset(G_, b, sh);
        }
#if REC_STATS
        if (G_.rank() == 0) atomicMax(&w.prof[P_R_WARPMAX], wsum);
#endif
    } else {
        GroupCTA G_;
        if (first >= total) return;
        ex_init(G_, b, sh);
        for (uint32_t item = first; item < total; item += stride) {
            uint2 x = w.ovf[item];
            bool ovf = false;
            extract_cg<GroupCTA, RowC>(G_, g, w, x.x, x.y, b, sh, &ovf);
#if REC_STATS
            if (G_.rank() == 0) atomicAdd(&w.prof[P_R_T1], 1ull);
#endif
            if (ovf && G_.rank() == 0) { sh.dirty = 1; push_overflow(w, 1, x); }
            G_.sync();
            ex_reset(G_, b, sh);
        }
    }
}

template <class RowC> __global__ void __launch_bounds__(256) k_extract_cg_big(GraphDev g, WsDev w) {
    __shared__ ExShared sh;
    GroupCTA G_;
    uint32_t n = min(w.ctr[C_NOVF2], w.ovf_cap);
    if (blockIdx.x >= n) return;
    ExBuf b = big_buf(w, blockIdx.x, sh);
    ex_init_clean(G_, sh);
    for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
        uint2 sc = w.ovf2[i];
        bool ovf = false;
        extract_cg<GroupCTA, RowC>(G_, g, w, sc.x, sc.y, b, sh, &ovf);
#if REC_STATS
        if (G_.rank() == 0) atomicAdd(&w.prof[P_R_T2], 1ull);
#endif
        if (ovf && G_.rank() == 0) { sh.dirty = 1; atomicOr(&w.st[sc.x].err, (uint32_t)E_EXTRACT); }
        G_.sync();
        ex_reset(G_, b, sh);
    }
}

// ====================================================================== run 2: attach, RPG, PTC
// Attach (R14): D_gi = min over V_C of h_m[v][i]; all finite -> RPG with S^m = max_i
// D_gi (Eq. 5) and S^r (Eq. 6).  One warp per candidate, byte-SIMD min over the V_C rows.
template <class RowM> __global__ void __launch_bounds__(256) k_attach(WsDev w) {
    typedef Row<RowM> R;
    const uint32_t lane = lane_id();
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    uint32_t total = w.coffs[w.nslots];
    for (uint32_t item = gw; item < total; item += nw) {
        uint32_t s = find_slot_warp(w.coffs, w.nslots, item);
        uint32_t c = item - w.coffs[s];
        SlotState &st = w.st[s];
        if (!st.in_phase) continue;
        Cand &cd = w.CD(s)[c];
        if (cd.attached) continue;
        const HV<RowM> H = w.Hs<RowM>(1, s);
        RowM mn = (RowM)~(RowM)0;
        for (uint32_t t = lane; t < cd.n_vc; t += 32) mn = vmin<RowM>(mn, R::load(H + w.arena[cd.vc_off + t]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mn = vmin<RowM>(mn, shfl(mn, lane ^ o));
        RowM used = used_mask<RowM>(st.T[1]);
        if ((R::eq(mn, R::splat(0xFF)) & used) == 0 && lane == 0) {
            uint32_t sm = R::maxb(mn & used);
            cd.sm = sm;
            cd.sr = rpg_score(st.gamma, cd.sc, sm);
            for (uint32_t i = 0; i < RIKI_MAX_TERMS; i++) cd.mdist[i] = i < st.T[1] ? R::byte(mn, i) : 0;
            cd.attached = 1;
            atomicAdd(&st.n_attached, 1u);
            if (w.bounded) {
                w.CST(s)[c] = 1;  // its RPG is recovered by a k_rpg_select wave if it can enter the top-k
            } else {
                uint32_t p = atomicAdd(&w.ctr[C_NNEWATT], 1u);
                w.newatt[p] = make_uint2(s, c);
            }
        }
    }
}

__device__ __forceinline__ uint32_t uf_find(volatile uint32_t *uf, uint32_t x) {
    while (true) {
        uint32_t p = uf[x];
        if (p == x) return x;
        x = p;
    }
}
__device__ __forceinline__ void uf_union(uint32_t *uf, uint32_t a, uint32_t b) {
    while (true) {
        a = uf_find(uf, a);
        b = uf_find(uf, b);
        if (a == b) return;
        if (a < b) { uint32_t t = a; a = b; b = t; }
        if (atomicCAS(&uf[a], a, b) == a) return;
    }
}

// RPG of an attached candidate: G^r = CG u (u_i SP(m_i, V_C)) recovered from the V_C nodes
// at distance D_gi (R18), then PTC (R19').
template <class G, class RowM> __device__ void extract_rpg(const G &G_, const GraphDev &g, const WsDev &w, uint32_t s,
                                                           uint32_t c, const ExBuf &b, ExShared &sh, bool *overflow) {
    typedef Row<RowM> R;
    SlotState &st = w.st[s];
    Cand &cd = w.CD(s)[c];
    const HV<RowM> H = w.Hs<RowM>(1, s);
    const uint32_t T = st.T[1];
    const bool blocking = T >= 2;
    if (cd.n_nodes > b.hu.items_cap || cd.n_nodes * 2 > b.hu.cap || cd.n_edges > b.cap_e) {
        *overflow = true;
        return;
    }
    for (uint32_t i = G_.rank(); i < cd.n_nodes; i += G_.size()) b.hu.insert(w.arena[cd.nodes_off + i], &sh.ovf);
    for (uint32_t i = G_.rank(); i < cd.n_edges; i += G_.size()) b.edges[i] = w.arena[cd.edges_off + i];
    if (G_.rank() == 0) sh.nedges = cd.n_edges;
    G_.sync();
    for (uint32_t j = 0; j < T && !sh.ovf; j++) {
        const uint32_t dj = cd.mdist[j];
        for (uint32_t t = G_.rank(); t < cd.n_vc; t += G_.size()) {
            uint32_t v = w.arena[cd.vc_off + t];
            if (R::byte(R::load(H + v), j) == dj) {
                int idx = b.hk.insert(v, &sh.ovf);
                if (idx >= 0) b.qh[idx] = (uint8_t)dj;
            }
        }
        G_.sync();
        if (!sh.ovf) bfs_column(G_, g, w, s, 1, j, H, blocking, b, sh);
        G_.sync();
        if (sh.ovf) break;
        ex_reset_hk(G_, b, sh);
    }
    G_.sync();
    if (sh.ovf) { *overflow = true; return; }
    *overflow = false;
    const uint32_t nn = min(sh.nu, b.hu.items_cap), ne = min(sh.nedges, b.cap_e);
    // ---- PTC: |M| = 1 trivial; else two distinct marginal keyword nodes X whose
    // every simple connection in G^r passes through V_C (endpoint-inclusive, R19').
    // ptc_mode 2 evaluates it on G^m only (nodes and edges of the marginal recovery);
    // ptc_mode 3 is SPEC's exclusive form (V_C-resident X never qualifies a pair).
    uint32_t pass = 1;
    if (T >= 2) {
        const int mode = st.ptc_mode;
        const uint32_t ncg = cd.n_edges;  // edges [0, ncg) are the CG's, [ncg, ne) G^m's
        RowM used = used_mask<RowM>(T);
        for (uint32_t i = G_.rank(); i < nn; i += G_.size()) {
            uint32_t sl = b.hu.slots[i];
            b.flag[sl] = mode == 2 ? 0 : 4;  // bit 4: node of the graph PTC is evaluated on
            b.uf[sl] = sl;
        }
        if (G_.rank() == 0) { sh.nx = 0; sh.xvc = 0; sh.mnr = EMPTY; sh.mxr = 0; }
        G_.sync();
        for (uint32_t t = G_.rank(); t < cd.n_vc; t += G_.size()) {
            uint32_t v = w.arena[cd.vc_off + t];
            int sl = b.hu.find(v);
            if (sl < 0) continue;
            b.flag[sl] |= 1;
            if (mode == 2) {  // recovery sources: V_C nodes at the marginal distance
                RowM r = R::load(H + v);
                for (uint32_t j = 0; j < T; j++)
                    if (R::byte(r, j) == cd.mdist[j]) b.flag[sl] |= 4;
            }
        }
        G_.sync();  // byte stores above must land before the word atomics below
        if (mode == 2) {
            for (uint32_t i = ncg + G_.rank(); i < ne; i += G_.size()) {
                uint32_t e = b.edges[i];
                int sa = b.hu.find(g.src[e]), sb = b.hu.find(g.dst[e]);
                if (sa >= 0) atomicOr((uint32_t *)&b.flag[sa & ~3] , 4u << (8 * (sa & 3)));
                if (sb >= 0) atomicOr((uint32_t *)&b.flag[sb & ~3], 4u << (8 * (sb & 3)));
            }
        }
        G_.sync();
        for (uint32_t i = G_.rank(); i < nn; i += G_.size()) {
            uint32_t sl = b.hu.slots[i];
            if (!(b.flag[sl] & 4)) continue;
            if (R::eq(R::load(H + b.hu.items[i]), 0) & used) {
                b.flag[sl] |= 2;
                atomicAdd(&sh.nx, 1u);
                if (b.flag[sl] & 1) sh.xvc = 1;
            }
        }
        G_.sync();
        if (sh.nx < 2) pass = 0;
        else if (mode != 3 && sh.xvc) pass = 1;
        else {
            for (uint32_t i = (mode == 2 ? ncg : 0) + G_.rank(); i < ne; i += G_.size()) {
                uint32_t e = b.edges[i];
                int sa = b.hu.find(g.src[e]), sb = b.hu.find(g.dst[e]);
                if (sa < 0 || sb < 0 || (b.flag[sa] & 1) || (b.flag[sb] & 1)) continue;
                if (!(b.flag[sa] & 4) || !(b.flag[sb] & 4)) continue;
                uf_union(b.uf, (uint32_t)sa, (uint32_t)sb);
            }
            G_.sync();
            for (uint32_t i = G_.rank(); i < nn; i += G_.size()) {
                uint32_t sl = b.hu.slots[i];
                if ((b.flag[sl] & 7) != 6) continue;  // X outside V_C, in the PTC graph
                uint32_t r = uf_find(b.uf, sl);
                atomicMin(&sh.mnr, r);
                atomicMax(&sh.mxr, r);
            }
            G_.sync();
            pass = sh.mnr != sh.mxr;
        }
    }
    G_.sync();
    // ---- write G^r lists
    if (G_.rank() == 0) sh.off = arena_alloc(w, nn + ne, s);
    G_.sync();
    const uint32_t off = sh.off;
    if (off != EMPTY) {
        for (uint32_t i = G_.rank(); i < nn; i += G_.size()) w.arena[off + i] = b.hu.items[i];
        for (uint32_t i = G_.rank(); i < ne; i += G_.size()) w.arena[off + nn + i] = b.edges[i];
    }
    G_.sync();
    if (G_.rank() == 0 && off != EMPTY) {
        cd.nodes_off = off; cd.n_nodes = nn;
        cd.edges_off = off + nn; cd.n_edges = ne;
        cd.ptc = pass;
        if (!pass) atomicAdd(&st.n_ptc_fail, 1u);
        if (pass || st.ptc_mode == 1) {
            uint32_t p = atomicAdd(&st.nR, 1u);
            if (p < w.capc) w.RK(s)[p] = rkey(cd.sr, cd.sc, cd.ext);
            else atomicOr(&st.err, (uint32_t)E_CAND);
        }
    }
}

template <class RowM, int TIER> __global__ void __launch_bounds__(tier_threads<TIER>()) k_extract_rpg(GraphDev g, WsDev w) {
    extern __shared__ __align__(16) uint8_t smx[];
    __shared__ ExShared shs[Tier<TIER>::GROUPS];
    const uint32_t n = TIER == 0 ? w.ctr[C_NNEWATT] : min(w.ctr[C_NOVF], w.ovf_cap);
    const uint32_t gi = TIER == 0 ? threadIdx.x >> 5 : 0;
    ExShared &sh = shs[gi];
    ExBuf b = smem_buf<TIER>(smx + smem_group<TIER>() * gi, sh);
    const uint32_t first = blockIdx.x * Tier<TIER>::GROUPS + gi, stride = gridDim.x * Tier<TIER>::GROUPS;
    if (TIER == 0) {
        GroupWarp G_;
        if (first >= n) return;
        ex_init(G_, b, sh);
        for (uint32_t i = first; i < n; i = rec_next(w, i, stride)) {
            uint2 sc = w.newatt[i];
            bool ovf = false;
            extract_rpg<GroupWarp, RowM>(G_, g, w, sc.x, sc.y, b, sh, &ovf);
            if (ovf && G_.rank() == 0) { sh.dirty = 1; push_overflow(w, 0, sc); }
            G_.sync();
            ex_reset(G_, b, sh);
        }
    } else {
        GroupCTA G_;
        if (first >= n) return;
        ex_init(G_, b, sh);
        for (uint32_t i = first; i < n; i += stride) {
            uint2 sc = w.ovf[i];
            bool ovf = false;
            extract_rpg<GroupCTA, RowM>(G_, g, w, sc.x, sc.y, b, sh, &ovf);
#if REC_STATS
            if (G_.rank() == 0) atomicAdd(&w.prof[P_R_T1RPG], 1ull);
#endif
            if (ovf && G_.rank() == 0) { sh.dirty = 1; push_overflow(w, 1, sc); }
            G_.sync();
            ex_reset(G_, b, sh);
        }
    }
}

template <class RowM> __global__ void __launch_bounds__(256) k_extract_rpg_big(GraphDev g, WsDev w) {
    __shared__ ExShared sh;
    GroupCTA G_;
    uint32_t n = min(w.ctr[C_NOVF2], w.ovf_cap);
    if (blockIdx.x >= n) return;
    ExBuf b = big_buf(w, blockIdx.x, sh);
    ex_init_clean(G_, sh);
    for (uint32_t i = blockIdx.x; i < n; i += gridDim.x) {
        uint2 sc = w.ovf2[i];
        bool ovf = false;
        extract_rpg<GroupCTA, RowM>(G_, g, w, sc.x, sc.y, b, sh, &ovf);
#if REC_STATS
        if (G_.rank() == 0) {
            atomicAdd(&w.prof[P_R_T2RPG], 1ull);
            atomicAdd(&w.prof[P_R_T2NODES], (unsigned long long)sh.nu);
            atomicAdd(&w.prof[P_R_T2EDGES], (unsigned long long)sh.nedges);
            atomicMax(&w.prof[P_R_T2MAXE], (unsigned long long)sh.nedges);
        }
#endif
        if (ovf && G_.rank() == 0) { sh.dirty = 1; atomicOr(&w.st[sc.x].err, (uint32_t)E_EXTRACT); }
        G_.sync();
        ex_reset(G_, b, sh);
    }
}

__global__ void k_reset_level_ctrs(WsDev w) {
    w.ctr[C_RECQ] = 0;
    w.ctr[C_NNEWATT] = 0;
    w.ctr[C_NOVF] = 0;
    w.ctr[C_NOVF2] = 0;
}

__device__ void cta_sort_u128(u128 *keys, uint32_t n, u128 *smem, uint32_t smem_cap) {
    if (n < 2) return;
    if (next_pow2(n) <= smem_cap) {
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) smem[i] = keys[i];
        __syncthreads();
        cta_bitonic_sort(smem, n);
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) keys[i] = smem[i];
        __syncthreads();
    } else {
        cta_bitonic_sort(keys, n);
    }
}

// Bounded RPG recovery (run 2, wave `last` = 0 or 1).  The answer is the k smallest keys
// (S^r, S^c, v) of the PTC-passing RPGs, and the k-th key of the results found so far (R)
// only decreases, so a candidate whose key is not below it can never enter the top-k: its
// RPG is not recovered (R21's argument for attached candidates).  The candidates attached at
// level l all have S^m = l, so their key order is their (S^c, v) order = candidate order.
// Wave 0 takes, per slot, the first k pending candidates (in order) that can still enter;
// wave 1 (after their PTC) takes every remaining one that still can.  One CTA per slot; the
// selected (slot, candidate) pairs go to the recovery tiers through the newatt list.  With the
// weight-sum tie-break (R29) every attached candidate is recovered (its key needs W).
__global__ void __launch_bounds__(256) k_rpg_select(WsDev w, uint32_t l_arg, int last) {
    const uint32_t l = l_arg == LV_DEVICE ? w.ctr[C_LEVEL] : l_arg;
    extern __shared__ __align__(16) u128 sm128[];
    __shared__ uint32_t taken, wcount[8];
    const uint32_t s = blockIdx.x;
    SlotState &st = w.st[s];
    if (!st.in_phase) return;
    uint32_t nR = min(st.nR, w.capc);
    if (last && nR != st.nR_sorted) {  // R gained the previous wave's results
        cta_sort_u128(w.RK(s), nR, sm128, U128_SORT_KEYS);
        if (threadIdx.x == 0) st.nR_sorted = nR;
    }
    const bool full = nR >= st.k && !st.tie_break;
    const u128 kth = full ? w.RK(s)[st.k - 1] : (u128)0;
    const uint32_t limit = last || st.tie_break ? 0xFFFFFFFFu : st.k;
    if (threadIdx.x == 0) taken = 0;
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    uint8_t *cst = w.CST(s);
    for (uint32_t c0 = 0; c0 < st.n_extract; c0 += blockDim.x) {
        const uint32_t c = c0 + threadIdx.x;
        bool pend = false;
        if (c < st.n_extract && cst[c] == 1) {
            const Cand &cd = w.CD(s)[c];
            if (cd.sm != l || (full && !(rkey(cd.sr, cd.sc, cd.ext) < kth))) cst[c] = 3;  // can never enter
            else pend = true;
        }
        const uint32_t b = __ballot_sync(FULLMASK, pend);
        if (lane == 0) wcount[wid] = __popc(b);
        __syncthreads();
        uint32_t before = taken;
        for (uint32_t i = 0; i < wid; i++) before += wcount[i];
        const uint32_t rank = before + __popc(b & lanemask_lt());
        if (pend && rank < limit) {
            cst[c] = 2;
            const uint32_t p = atomicAdd(&w.ctr[C_NNEWATT], 1u);
            w.newatt[p] = make_uint2(s, c);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t t = 0;
            for (uint32_t i = 0; i < blockDim.x / 32; i++) t += wcount[i];
            taken += t;
        }
        __syncthreads();
        if (taken >= limit) break;
    }
}

// Termination of run 2 at level l (after attach): depth, empty frontier, all attached, or
// the exact bound (R21): |R| >= k and the best key any unattached candidate can still
// reach, (gamma*S^c + (1-gamma)*(l+1), S^c, v), is worse than the k-th key of R.
__global__ void k_decide_m(WsDev w, uint32_t l_arg) {
    const uint32_t l = l_arg == LV_DEVICE ? w.ctr[C_LEVEL] : l_arg;
    extern __shared__ __align__(16) u128 sm128[];
    __shared__ uint32_t first;
    uint32_t s = blockIdx.x;
    SlotState &st = w.st[s];
    if (!st.in_phase) return;
    if (threadIdx.x == 0) first = EMPTY;
    __syncthreads();
    uint32_t nR = min(st.nR, w.capc);
    if (nR != st.nR_sorted) cta_sort_u128(w.RK(s), nR, sm128, U128_SORT_KEYS);  // only when new RPGs arrived
    // attachment is monotone, so the first unattached candidate only moves forward
    const uint32_t c_begin = st.first_unatt, c_end = st.n_extract;
    for (uint32_t c0 = c_begin; c0 < c_end; c0 += blockDim.x) {
        uint32_t c = c0 + threadIdx.x;
        if (c < c_end && !w.CD(s)[c].attached) atomicMin(&first, c);
        __syncthreads();
        const bool found = first != EMPTY;  // uniform: read between two barriers
        __syncthreads();
        if (found) break;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        st.nR_sorted = nR;
        st.first_unatt = first == EMPTY ? st.n_extract : first;
    }
    if (threadIdx.x == 0) {
        bool stop = l >= st.depth || st.nq[l & 1] == 0 || first == EMPTY;
        if (!stop && st.early_term != 2 && nR >= st.k) {
            const Cand &fu = w.CD(s)[first];
            const u128 kth = w.RK(s)[st.k - 1];
            if (st.early_term == 0) {
                u128 best = rkey(rpg_score(st.gamma, fu.sc, l + 1), fu.sc, fu.ext);
                // tie-break (R29): a candidate's W is unknown until it attaches, so only a
                // strictly larger (S^r, S^c) excludes it
                stop = st.tie_break ? (kth >> 32) < (best >> 32) : kth < best;
            } else {  // paper-literal inequality (Theorem earlyTermination)
                uint64_t ck = (uint64_t)kth;  // (S^c << 32 | v) locates the k-th RPG's candidate
                uint32_t lo = 0, hi = st.n_extract;
                const uint64_t *K = w.CK(s);
                while (lo < hi) { uint32_t m = (lo + hi) >> 1; if (K[m] < ck) lo = m + 1; else hi = m; }
                const Cand &kc = w.CD(s)[lo];
                double rhs = rpg_score(st.gamma, fu.sc, kc.sm);  // gamma*min S^c + (1-gamma)*S^m(kth)
                stop = kc.sr <= rhs;
            }
        }
        st.stop_m = stop;
    }
}

// ====================================================================== finalize
__global__ void k_final_select(WsDev w) {
    extern __shared__ __align__(16) u128 sm128[];
    uint32_t s = blockIdx.x;
    SlotState &st = w.st[s];
    if (!st.active || st.err) {
        if (threadIdx.x == 0) st.nres = 0;
        return;
    }
    if (st.T[1] == 0 && st.tie_break) {  // M = empty with the tie-break: rank the CGs as keys
        for (uint32_t i = threadIdx.x; i < st.n_extract; i += blockDim.x) {
            const Cand &cd = w.CD(s)[i];
            w.RK(s)[i] = rkey((double)cd.sc, cd.sc, cd.ext);  // already in (S^c, v) order
        }
        if (threadIdx.x == 0) st.nR = st.n_extract;
        __syncthreads();
    } else if (st.T[1] == 0) {  // M = empty: top-k CGs by (S^c, v)
        uint32_t n = min(st.k, st.n_extract);
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) w.resid[(size_t)s * w.kmax + i] = i;
        if (threadIdx.x == 0) st.nres = n;
        return;
    }
    uint32_t nR = min(st.nR, w.capc);
    cta_sort_u128(w.RK(s), nR, sm128, U128_SORT_KEYS);
    uint32_t n = min(st.k, nR);
    if (st.tie_break) {  // R29: the order of [0, end of the k-th key's (S^r, S^c) group) needs W
        if (threadIdx.x == 0) {
            uint32_t e = n;
            if (n) {
                const u128 g = w.RK(s)[n - 1] >> 32;
                while (e < nR && (w.RK(s)[e] >> 32) == g) e++;
            }
            st.ntie = e;
            st.nres = n;
        }
        return;  // k_tie_weights + k_tie_select finish the selection
    }
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        u128 key = w.RK(s)[i];
        uint64_t ck = (uint64_t)key;  // (sc << 32 | v)
        uint32_t lo = 0, hi = st.n_extract;
        const uint64_t *K = w.CK(s);
        while (lo < hi) { uint32_t m = (lo + hi) >> 1; if (K[m] < ck) lo = m + 1; else hi = m; }
        w.resid[(size_t)s * w.kmax + i] = lo;
    }
    if (threadIdx.x == 0) st.nres = n;
}

// Candidate index of an (S^r, S^c, v) key: CK is sorted by (S^c << 32 | caller id).
__device__ __forceinline__ uint32_t cand_of_key(const WsDev &w, const SlotState &st, uint32_t s, u128 key) {
    const uint64_t ck = (uint64_t)key;
    uint32_t lo = 0, hi = st.n_extract;
    const uint64_t *K = w.CK(s);
    while (lo < hi) { uint32_t m = (lo + hi) >> 1; if (K[m] < ck) lo = m + 1; else hi = m; }
    return lo;
}

// Tie-break (R29): W = sum of round(w * 2^32) over the DISTINCT edges of each result
// in [0, ntie) (its edge list may repeat an edge shared by the CG and G^m) -- or, with
// cgs = true, of every recovered candidate CG of a beam_mode-1 slot.  Block per item: the
// list is sorted in shared memory (arena for long lists), then reduced.
__global__ void __launch_bounds__(256) k_tie_weights(GraphDev g, WsDev w, bool cgs) {
    extern __shared__ __align__(16) uint32_t sm32[];
    __shared__ unsigned long long acc;
    __shared__ uint32_t s_buf;
    const uint32_t s = blockIdx.y;
    const SlotState &st = w.st[s];
    if (!st.active || st.err || !st.tie_break || (cgs && st.beam_mode != 1)) return;
    const uint32_t nitems = cgs ? st.n_extract : st.ntie;
    for (uint32_t i = blockIdx.x; i < nitems; i += gridDim.x) {
        const uint32_t c = cgs ? i : cand_of_key(w, st, s, w.RK(s)[i]);
        Cand &cd = w.CD(s)[c];
        const uint32_t n = cd.n_edges;
        uint32_t *buf = sm32;
        if (next_pow2(n) > SORT_SMEM) {
            if (threadIdx.x == 0) s_buf = arena_alloc(w, next_pow2(n), s);
            __syncthreads();
            if (s_buf == EMPTY) return;  // E_ARENA raised: the batch is re-run with a larger arena
            buf = w.arena + s_buf;
        }
        if (threadIdx.x == 0) acc = 0;
        for (uint32_t j = threadIdx.x; j < n; j += blockDim.x) buf[j] = w.arena[cd.edges_off + j];
        __syncthreads();
        cta_bitonic_sort(buf, n);
        unsigned long long part = 0;
        for (uint32_t j = threadIdx.x; j < n; j += blockDim.x)
            if (j == 0 || buf[j] != buf[j - 1]) part += g.wfix[buf[j]];
        atomicAdd(&acc, part);
        __syncthreads();
        if (threadIdx.x == 0) cd.wsum = acc;
        __syncthreads();
    }
}

// Beam of width w with the tie-break (R29): keep the w smallest (S^c, W(CG), v) of the
// recovered tie-kept candidates, compacted in (S^c, v) order (candidate index order).
// RK is free before run 2 and serves as sort space.
__global__ void k_beam_tie(WsDev w) {
    extern __shared__ __align__(16) u128 sm128[];
    const uint32_t s = blockIdx.x;
    SlotState &st = w.st[s];
    if (!st.active || st.err || !st.tie_break || st.beam_mode != 1) return;
    const uint32_t n = st.n_extract, keep = min(n, st.w);
    if (n > keep) {
        u128 *K = w.RK(s);
        Cand *CD = w.CD(s);
        uint64_t *CK = w.CK(s);
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x)
            K[i] = (u128)CD[i].sc << 96 | (u128)CD[i].wsum << 32 | i;
        __syncthreads();
        cta_sort_u128(K, n, sm128, U128_SORT_KEYS);
        for (uint32_t i = threadIdx.x; i < keep; i += blockDim.x) K[i] = (uint32_t)K[i];
        __syncthreads();
        cta_sort_u128(K, keep, sm128, U128_SORT_KEYS);  // kept indices ascending = (S^c, v) order
        // compaction in place: source index K[j] >= j; chunk reads happen before chunk writes
        for (uint32_t j0 = 0; j0 < keep; j0 += blockDim.x) {
            const uint32_t j = j0 + threadIdx.x;
            Cand cd;
            uint64_t ck = 0;
            if (j < keep) { cd = CD[(uint32_t)K[j]]; ck = CK[(uint32_t)K[j]]; }
            __syncthreads();
            if (j < keep) { CD[j] = cd; CK[j] = ck; }
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) {
        st.n_extract = keep;
        st.ncand_kept = keep;
    }
}

// Tie-break order: every tie group (equal (S^r, S^c)) of [0, ntie) re-sorted by (W, v); the
// sort key is (group start << 96 | W << 32 | candidate index) -- within a group S^c is fixed,
// so candidate index order is caller-id order.
__global__ void k_tie_select(WsDev w) {
    extern __shared__ __align__(16) u128 sm128[];
    const uint32_t s = blockIdx.x;
    const SlotState &st = w.st[s];
    if (!st.active || st.err || !st.tie_break) return;
    const uint32_t nt = st.ntie;
    uint2 *T = w.tie + (size_t)s * w.capc;
    u128 *K = w.RK(s);
    for (uint32_t i = threadIdx.x; i < nt; i += blockDim.x) {
        const u128 key = K[i], grp = key >> 32;
        uint32_t lo = 0, hi = i;  // first index of i's group
        while (lo < hi) { uint32_t m = (lo + hi) >> 1; if ((K[m] >> 32) < grp) lo = m + 1; else hi = m; }
        T[i] = make_uint2(cand_of_key(w, st, s, key), lo);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < nt; i += blockDim.x) {
        const uint2 t = T[i];
        K[i] = (u128)t.y << 96 | (u128)w.CD(s)[t.x].wsum << 32 | t.x;
    }
    __syncthreads();
    cta_sort_u128(K, nt, sm128, U128_SORT_KEYS);
    for (uint32_t i = threadIdx.x; i < st.nres; i += blockDim.x) w.resid[(size_t)s * w.kmax + i] = (uint32_t)K[i];
}

// sort + unique a u32 list into the output buffer; returns (offset, count) via sh
__device__ void sort_unique_out(const WsDev &w, uint32_t s, const uint32_t *src, uint32_t n, const uint32_t *map,
                                uint32_t *smem, uint32_t *scan, uint32_t *res_off, uint32_t *res_n) {
    __shared__ uint32_t s_off, s_buf;
    uint32_t *buf = smem;
    bool global = next_pow2(n) > SORT_SMEM;
    if (global) {
        if (threadIdx.x == 0) s_buf = arena_alloc(w, next_pow2(n), s);
        __syncthreads();
        if (s_buf == EMPTY) { *res_off = 0; *res_n = 0; return; }
        buf = w.arena + s_buf;
    }
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) buf[i] = map ? map[src[i]] : src[i];
    __syncthreads();
    cta_bitonic_sort(buf, n);
    // unique: per-thread contiguous chunk counts + block scan
    uint32_t per = (n + blockDim.x - 1) / blockDim.x;
    uint32_t b0 = min(threadIdx.x * per, n), b1 = min(b0 + per, n);
    uint32_t cnt = 0;
    for (uint32_t i = b0; i < b1; i++) cnt += (i == 0 || buf[i] != buf[i - 1]);
    scan[threadIdx.x] = cnt;
    __syncthreads();
    for (uint32_t o = 1; o < blockDim.x; o <<= 1) {
        uint32_t v = threadIdx.x >= o ? scan[threadIdx.x - o] : 0;
        __syncthreads();
        scan[threadIdx.x] += v;
        __syncthreads();
    }
    uint32_t total = scan[blockDim.x - 1];
    if (threadIdx.x == 0) {
        unsigned long long p = atomicAdd(w.out_used, (unsigned long long)total);
        if (p + total > w.out_cap) { atomicOr(&w.st[s].err, (uint32_t)E_OUT); s_off = EMPTY; }
        else s_off = (uint32_t)p;
    }
    __syncthreads();
    uint32_t off = s_off;
    if (off != EMPTY) {
        uint32_t pos = off + scan[threadIdx.x] - cnt;
        for (uint32_t i = b0; i < b1; i++)
            if (i == 0 || buf[i] != buf[i - 1]) w.out[pos++] = buf[i];
    }
    __syncthreads();
    *res_off = off;
    *res_n = total;
}

template <class RowC> __global__ void __launch_bounds__(256) k_final_lists(GraphDev g, WsDev w) {
    extern __shared__ __align__(16) uint32_t sm32[];
    __shared__ uint32_t scan[256];
    uint32_t r = blockIdx.x, s = blockIdx.y;
    const SlotState &st = w.st[s];
    if (r >= st.nres) return;
    uint32_t c = w.resid[(size_t)s * w.kmax + r];
    const Cand &cd = w.CD(s)[c];
    OutHdr h;
    memset(&h, 0, sizeof(h));
    h.central = cd.ext;
    h.sc = cd.sc;
    h.sm = st.T[1] ? cd.sm : 0;
    h.ptc = cd.ptc;
    h.score = st.T[1] ? cd.sr : (double)cd.sc;
    sort_unique_out(w, s, w.arena + cd.nodes_off, cd.n_nodes, g.iperm, sm32, scan, &h.nodes_off, &h.n_nodes);
    sort_unique_out(w, s, w.arena + cd.edges_off, cd.n_edges, nullptr, sm32, scan, &h.edges_off, &h.n_edges);
    sort_unique_out(w, s, w.arena + cd.vc_off, cd.n_vc, g.iperm, sm32, scan, &h.vc_off, &h.n_vc);
    RowC hv = Row<RowC>::load(w.Hs<RowC>(0, s) + cd.v);
    for (uint32_t j = 0; j < RIKI_MAX_TERMS; j++) {
        h.cdist[j] = j < st.T[0] ? Row<RowC>::byte(hv, j) : 0;
        h.mdist[j] = j < st.T[1] ? cd.mdist[j] : 0;
    }
    if (threadIdx.x == 0) w.hdr[(size_t)s * w.kmax + r] = h;
}

// ====================================================================== debug boundary
template <class RowT>
__global__ void k_pack_H(GraphDev g, WsDev w, uint32_t T, uint8_t *Hout, uint8_t *blk, int blocking) {
    const HV<RowT> H = w.Hs<RowT>(0, 0);
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < w.V; v += gridDim.x * blockDim.x) {
        RowT r = Row<RowT>::load(H + g.perm[v]);  // output indexed by caller id
        for (uint32_t j = 0; j < T; j++) Hout[(size_t)v * T + j] = (uint8_t)Row<RowT>::byte(r, j);
        blk[v] = (blocking && Row<RowT>::eq(r, Row<RowT>::splat(0xFF)) == 0) ? (uint8_t)Row<RowT>::maxb(r) : 0xFF;
    }
}

}  // namespace

// ====================================================================== host side
struct Workspace {
    uint32_t track_reached = 0;
    uint32_t tie_break = 0;  // current batch uses the weight-sum tie-break (R29)
    uint32_t beam_tie = 0;   // ... with beam_mode 1 (beam truncated by W(CG))
    uint32_t hnode = 0, SP = 0;  // H layout of the current batch
    uint32_t hcap[2] = {0, 0};   // bytes per H row allocated per run
    uint32_t cur = 0;  // slots used by the current batch (<= slots)
    uint32_t slots = 0, V = 0, W = 0, capc = 0, kmax = 0, heavy_cap = 0, ovf_cap = 0, big_ctas = 0;
    uint64_t arena_cap = 0, out_cap = 0, big_words = 0;
    uint8_t *H[2] = {nullptr, nullptr};
    uint32_t qcap = 0;  // entries per level queue
    unsigned long long *offs = nullptr;
    uint32_t *q = nullptr, *bm = nullptr, *jq = nullptr, *jbm = nullptr, *coffs = nullptr, *pslots = nullptr, *ppos = nullptr, *ctr = nullptr, *arena = nullptr,
             *big = nullptr, *resid = nullptr, *out = nullptr;
    uint4 *mtab = nullptr;
    uint64_t *ck = nullptr, *ck2 = nullptr;  // candidate keys; ck2 = sorted copy (segmented radix sort)
    int *seg_b = nullptr, *seg_e = nullptr;
    void *sort_tmp = nullptr;
    size_t sort_tmp_bytes = 0;
    uint32_t sort_group = 1;  // slots per segmented-sort call (item counts stay int-sized)
    Cand *cd = nullptr;
    u128 *rk = nullptr;
    SlotState *st = nullptr;
    uint4 *heavy = nullptr;
    unsigned long long *prof = nullptr, *arena_used = nullptr, *out_used = nullptr;
    uint2 *newatt = nullptr, *ovf = nullptr, *ovf2 = nullptr, *tie = nullptr;
    uint8_t *cst = nullptr;
    uint32_t bounded = 0;
    OutHdr *hdr = nullptr;
    uint32_t *h_ctr = nullptr;  // pinned
    uint64_t bytes = 0;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    std::vector<cudaEvent_t> evpool;
    // CUDA graphs of LEVEL_BATCH-level chunks of the level loop, keyed by everything their
    // kernel nodes bake in (phase, first level, kernel variants, grids, device views)
    struct GraphEntry {
        std::vector<uint8_t> key;
        cudaGraphExec_t exec;
        uint32_t kernels;
    };
    std::vector<GraphEntry> gcache;
    void clear_graphs() {
        for (GraphEntry &e : gcache) cudaGraphExecDestroy(e.exec);
        gcache.clear();
    }
    cudaEvent_t event(uint32_t i) {
        while (evpool.size() <= i) {
            cudaEvent_t e;
            CUDA_TRY(cudaEventCreate(&e));
            evpool.push_back(e);
        }
        return evpool[i];
    }
    // state of the last device batch (for engine_fetch)
    uint32_t last_n = 0;
    std::vector<uint32_t> last_map;  // slot -> query index of the last batch
    int last_rb[2] = {4, 4};
    std::vector<std::vector<riki_results *>> dummy;
    std::vector<void *> allocs;

    template <class T> T *alloc(size_t n) {
        T *p = nullptr;
        if (n == 0) n = 1;
        if (cudaMalloc(&p, n * sizeof(T)) != cudaSuccess) {
            cudaGetLastError();
            RIKI_THROW(RIKI_ENOMEM, "workspace cudaMalloc of " + std::to_string(n * sizeof(T)) + " bytes failed");
        }
        allocs.push_back(p);
        bytes += n * sizeof(T);
        return p;
    }
    void release() {
        clear_graphs();
        for (void *p : allocs) cudaFree(p);
        allocs.clear();
        if (h_ctr) cudaFreeHost(h_ctr);
        h_ctr = nullptr;
        if (ev0) cudaEventDestroy(ev0);
        if (ev1) cudaEventDestroy(ev1);
        ev0 = ev1 = nullptr;
        for (cudaEvent_t e : evpool) cudaEventDestroy(e);
        evpool.clear();
        bytes = 0;
    }
    WsDev dev() const {
        WsDev d;
        memset(&d, 0, sizeof(d));  // padding too: the struct is part of CUDA-graph cache keys
        d.st = st; d.nslots = cur ? cur : slots; d.V = V; d.W = W; d.capc = capc; d.kmax = kmax;
        d.H[0] = H[0]; d.H[1] = H[1]; d.hnode = hnode; d.SP = SP; d.rb[0] = last_rb[0]; d.rb[1] = last_rb[1];
        d.q = q; d.qcap = qcap; d.bm = bm; d.jq = jq; d.jbm = jbm; d.ck = ck; d.cd = cd; d.rk = rk; d.offs = offs; d.coffs = coffs; d.pslots = pslots; d.ppos = ppos; d.track_reached = track_reached;
        d.heavy = heavy; d.heavy_cap = heavy_cap; d.ctr = ctr; d.prof = prof;
        d.arena = arena; d.arena_used = arena_used; d.arena_cap = arena_cap;
        d.newatt = newatt; d.ovf = ovf; d.ovf2 = ovf2; d.ovf_cap = ovf_cap; d.cst = cst; d.bounded = bounded;
        d.big = big; d.big_words = big_words; d.mtab = mtab;
        d.hdr = hdr; d.tie = tie; d.resid = resid; d.out = out; d.out_used = out_used; d.out_cap = out_cap;
        return d;
    }
};

namespace {

struct Tracer {  // RIKI_TRACE=<ms>: print the stage times of calls slower than <ms>
    double thr = getenv("RIKI_TRACE") ? atof(getenv("RIKI_TRACE")) : -1;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now(), t = t0;
    std::string log;
    void operator()(const char *what) {
        if (thr < 0) return;
        auto n = std::chrono::steady_clock::now();
        char b[96];
        snprintf(b, sizeof b, " %s=%.3f", what, std::chrono::duration<double, std::milli>(n - t).count());
        log += b;
        t = n;
    }
    ~Tracer() {
        if (thr < 0) return;
        double tot = std::chrono::duration<double, std::milli>(t - t0).count();
        if (tot >= thr) fprintf(stderr, "[riki] %.3f ms:%s\n", tot, log.c_str());
    }
};

// NVTX ranges (header-only NVTX v3: no-ops unless a profiler such as Nsight Systems is attached):
// one per section of a batch (central run, CG recovery, marginal run, finalize) and, in the
// plain-launch path, one per level.  begin() closes the open range first.
struct Nvtx {
    bool open = false;
    void begin(const char *m) {
        end();
        nvtxRangePushA(m);
        open = true;
    }
    void end() {
        if (open) nvtxRangePop();
        open = false;
    }
    ~Nvtx() { end(); }
};

struct Caps {
    uint32_t slots, capc, kmax, qcap;
    uint64_t arena, out;
    uint32_t rb[2];  // bytes per H row needed by each run
};

constexpr uint64_t ARENA_MAX_WORDS = 0xFFFFFF00ull;  // largest arena addressable by u32 offsets


void ensure_workspace(riki_graph *g, const Caps &c) {
    Workspace *ws = g->ws;
    if (ws && ws->slots >= c.slots && ws->V == g->V && ws->capc >= c.capc && ws->kmax >= c.kmax &&
        ws->arena_cap >= c.arena && ws->out_cap >= c.out && ws->hcap[0] >= c.rb[0] && ws->hcap[1] >= c.rb[1] &&
        ws->qcap >= c.qcap)
        return;
    uint32_t hb0 = std::max<uint32_t>(c.rb[0], ws ? ws->hcap[0] : 0), hb1 = std::max<uint32_t>(c.rb[1], ws ? ws->hcap[1] : 0);
    if (ws) { ws->release(); delete ws; g->ws = nullptr; }
    g->stats.reallocs++;
    if (getenv("RIKI_TRACE"))
        fprintf(stderr, "[riki] workspace: slots %u capc %u kmax %u qcap %u arena %llu words out %llu rb %u/%u\n", c.slots,
                c.capc, c.kmax, c.qcap, (unsigned long long)c.arena, (unsigned long long)c.out, c.rb[0], c.rb[1]);
    ws = new Workspace();
    g->ws = ws;
    const uint32_t V = g->V;
    ws->slots = c.slots; ws->V = V; ws->W = (V + 31) / 32; ws->capc = c.capc; ws->kmax = c.kmax;
    ws->arena_cap = c.arena; ws->out_cap = c.out;
    const size_t S = c.slots;
    ws->hcap[0] = hb0;
    ws->hcap[1] = hb1;
    const size_t SG = std::max<size_t>(8, HGRP);  // node-major / grouped layouts pad the slots
    const size_t S8 = (S + SG - 1) / SG * SG;
    ws->H[0] = ws->alloc<uint8_t>(S8 * V * hb0);
    ws->H[1] = ws->alloc<uint8_t>(S8 * V * hb1);
    ws->qcap = c.qcap;
    ws->q = ws->alloc<uint32_t>(S * 2 * (size_t)c.qcap);
    ws->jq = ws->alloc<uint32_t>(2 * (size_t)V);
    ws->jbm = ws->alloc<uint32_t>(2 * (size_t)ws->W);
    CUDA_TRY(cudaMemset(ws->jbm, 0, 2 * (size_t)ws->W * 4));
    ws->ck = ws->alloc<uint64_t>(S * c.capc);
    ws->ck2 = ws->alloc<uint64_t>(S * c.capc);
    ws->seg_b = ws->alloc<int>(S + 1);
    ws->seg_e = ws->alloc<int>(S + 1);
    ws->sort_group = (uint32_t)std::max<size_t>(1, std::min<size_t>(S, (1ull << 30) / c.capc));
    CUDA_TRY(cub::DeviceSegmentedRadixSort::SortKeys(nullptr, ws->sort_tmp_bytes, (const unsigned long long *)ws->ck,
                                                     (unsigned long long *)ws->ck2, (int)(ws->sort_group * (size_t)c.capc),
                                                     (int)ws->sort_group, ws->seg_b, ws->seg_e, 0, 40));
    ws->sort_tmp = ws->alloc<uint8_t>(ws->sort_tmp_bytes);
    ws->cd = ws->alloc<Cand>(S * c.capc);
    ws->rk = ws->alloc<u128>(S * c.capc);
    ws->st = ws->alloc<SlotState>(S);
    ws->offs = ws->alloc<unsigned long long>(S + 1);
    ws->coffs = ws->alloc<uint32_t>(S + 1);
    ws->pslots = ws->alloc<uint32_t>(S + 1);
    ws->ppos = ws->alloc<uint32_t>(S + 1);
    uint64_t hc = (uint64_t)S * (g->E / CHUNK + g->E / HEAVY + 64);
    ws->heavy_cap = (uint32_t)std::min<uint64_t>(hc, 1u << 28);
    ws->heavy = ws->alloc<uint4>(ws->heavy_cap);
    ws->ctr = ws->alloc<uint32_t>(C_NCTR);
    ws->prof = ws->alloc<unsigned long long>(P_NPROF);
    ws->arena = ws->alloc<uint32_t>(c.arena);
    ws->arena_used = ws->alloc<unsigned long long>(1);
    ws->newatt = ws->alloc<uint2>(S * c.capc);
    ws->cst = ws->alloc<uint8_t>(S * c.capc);
    ws->ovf_cap = (uint32_t)(S * c.capc);
    ws->ovf = ws->alloc<uint2>(ws->ovf_cap);
    ws->ovf2 = ws->alloc<uint2>(ws->ovf_cap);
    ws->big_ctas = V <= (4u << 20) ? 8 : 2;
    if (const char *e = getenv("RIKI_BIG_CTAS")) ws->big_ctas = std::max(1, atoi(e));  // A/B
    uint64_t cu = next_pow2(2 * V + 2);
    ws->big_words = cu * 3 + 4ull * (V + 1) + cu / 4 + (V + 1) / 4 + 32 + std::max<uint64_t>(std::min<uint64_t>(g->E, 1ull << 26), 1u << 20);
    ws->mtab = ws->alloc<uint4>(S * 16 * MAPCAP);
    ws->big = ws->alloc<uint32_t>(ws->big_words * ws->big_ctas);
    CUDA_TRY(cudaMemset(ws->big, 0xFF, ws->big_words * ws->big_ctas * 4));  // EMPTY tables (ex_init_clean)
    ws->hdr = ws->alloc<OutHdr>(S * c.kmax);
    ws->resid = ws->alloc<uint32_t>(S * c.kmax);
    ws->tie = ws->alloc<uint2>(S * c.capc);
    ws->out = ws->alloc<uint32_t>(c.out);
    ws->out_used = ws->alloc<unsigned long long>(1);
    CUDA_TRY(cudaMallocHost(&ws->h_ctr, 64 * sizeof(uint32_t)));
    CUDA_TRY(cudaEventCreate(&ws->ev0));
    CUDA_TRY(cudaEventCreate(&ws->ev1));
    // function attributes are per device: set them once on every device a graph lives on
    static std::atomic<uint64_t> attr_done{0};
    const uint64_t dbit = 1ull << (g->device & 63);
    if (!(attr_done.load() & dbit)) {
#define SET_EX_ATTR(K) CUDA_TRY(cudaFuncSetAttribute(K<uint32_t, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_ex<1>())); \
        CUDA_TRY(cudaFuncSetAttribute(K<uint64_t, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_ex<1>())); \
        CUDA_TRY(cudaFuncSetAttribute(K<uint16_t, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_ex<1>()));
        SET_EX_ATTR(k_extract_cg)
        SET_EX_ATTR(k_extract_rpg)
#undef SET_EX_ATTR
        CUDA_TRY(cudaFuncSetAttribute(k_decide_m, cudaFuncAttributeMaxDynamicSharedMemorySize, U128_SORT_KEYS * 16));
        CUDA_TRY(cudaFuncSetAttribute(k_rpg_select, cudaFuncAttributeMaxDynamicSharedMemorySize, U128_SORT_KEYS * 16));
        CUDA_TRY(cudaFuncSetAttribute(k_final_select, cudaFuncAttributeMaxDynamicSharedMemorySize, U128_SORT_KEYS * 16));
        CUDA_TRY(cudaFuncSetAttribute(k_tie_select, cudaFuncAttributeMaxDynamicSharedMemorySize, U128_SORT_KEYS * 16));
        CUDA_TRY(cudaFuncSetAttribute(k_beam_tie, cudaFuncAttributeMaxDynamicSharedMemorySize, U128_SORT_KEYS * 16));
        CUDA_TRY(cudaFuncSetAttribute(k_tie_weights, cudaFuncAttributeMaxDynamicSharedMemorySize, SORT_SMEM * 4));
        CUDA_TRY(cudaFuncSetAttribute(k_final_lists<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, SORT_SMEM * 4));
        CUDA_TRY(cudaFuncSetAttribute(k_final_lists<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, SORT_SMEM * 4));
        CUDA_TRY(cudaFuncSetAttribute(k_final_lists<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, SORT_SMEM * 4));
        attr_done.fetch_or(dbit);
    }
}

unsigned grid_of(uint64_t work, unsigned per_block, unsigned cap = 148 * 16) {
    uint64_t b = (work + per_block - 1) / per_block;
    return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(b, cap));
}

struct Launch {
    riki_graph *g;
    cudaStream_t s;
    uint64_t launches = 0;
    double expand_ms = 0;
    uint64_t expand_launches = 0;
    uint32_t nev = 0;                 // profiling events recorded (pairs around each expansion)
    double sec_ms[4] = {0, 0, 0, 0};  // central run, recovery, marginal run, finalize (host wall between syncs)
    uint64_t levels = 0;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    void mark(int sec) {
        auto t = std::chrono::steady_clock::now();
        sec_ms[sec] += std::chrono::duration<double, std::milli>(t - t0).count();
        t0 = t;
    }
    void check(int line) {
        cudaError_t e = cudaGetLastError();
        static const bool sync_each = getenv("RIKI_SYNC") != nullptr;  // diagnostics: fault -> launch site
        if (e == cudaSuccess && sync_each) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess)
            RIKI_THROW(RIKI_ECUDA, std::string("kernel launch (engine.cu:") + std::to_string(line) + "): " + cudaGetErrorString(e));
        launches++;
    }
};

// Resident tier-0 recovery blocks per SM (one full wave), from the occupancy calculator.
template <class K> uint32_t tier0_blocks_per_sm(K kernel) {
    static uint32_t cached = 0;  // per kernel instantiation
    if (!cached) {
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kernel, tier_threads<0>(), smem_ex<0>()) != cudaSuccess || nb < 1)
            nb = 1;
        cached = (uint32_t)nb;
    }
    return cached;
}

// Device-side loop control of the whole-run graph (after level l's plan and expansion):
// continue while some slot is still in its run and l < max_levels (the host loop's rule),
// and advance the level counter.
__global__ void k_loop_cond(WsDev w, cudaGraphConditionalHandle h, uint32_t max_levels) {
    const uint32_t l = w.ctr[C_LEVEL];
    const bool go = w.ctr[C_ACTIVE] != 0 && l < max_levels;
    w.ctr[C_LEVEL] = l + 1;
    cudaGraphSetConditional(h, go ? 1u : 0u);
}

// One level's push expansion (light items, then the heavy chunks), one wave of blocks each.
template <class RowT, bool CNT, bool BIG>
void expand_launch(Launch &L, const GraphDev &gd, const WsDev &wd, int ph, uint32_t l, bool wide) {
    constexpr unsigned grid = 148 * ExpMinB<RowT, BIG>::v;
    if (wide)
        k_expand<RowT, true, false, CNT, BIG><<<grid, 256, 0, L.s>>>(gd, wd, ph, l);
    else
        k_expand<RowT, false, false, CNT, BIG><<<grid, 256, 0, L.s>>>(gd, wd, ph, l);
    L.check(__LINE__);
    k_expand_heavy<RowT, false, CNT, BIG><<<grid, 256, 0, L.s>>>(gd, wd, ph, l);
    L.check(__LINE__);
}

// One vertex-partitioned level: pull over this rank's node range into its
// slice of the bit-plane buffer (every range, in simulated mode), one in-place all-gather
// on the search stream, then every rank applies all slices.  Identical H, blocks, frontiers
// and candidates on every rank, so termination needs no further collective.
template <class RowT>
void vp_level(Launch &L, const GraphDev &gd, const WsDev &wd, int ph, uint32_t l, uint32_t npull) {
    DistState *d = L.g->dist;
    cudaStream_t s = L.s;
    const size_t chunk = (size_t)npull * sizeof(RowT) * d->wc;
    uint32_t *x = dist_exchange_buffer(L.g, chunk);
    CUDA_TRY(cudaMemsetAsync(x, 0, chunk * 4 * d->nranks, s));
    for (int r = 0; r < d->nranks; r++) {
        if (!d->simulated && r != d->rank) continue;
        const uint32_t lo = d->bounds[r], hi = d->bounds[r + 1];
        if (hi <= lo) continue;
        const uint32_t hh = std::min(hi, gd.Vh);
        const uint32_t nbh = hh > lo ? std::min<uint32_t>((hh - lo + 7) / 8, 148 * 8) : 0;
        const uint32_t ll = std::max(lo, gd.Vh);
        const uint32_t nbl = hi > ll ? std::min<uint32_t>((hi - ll + 255) / 256, 148 * 8) : 0;
        k_pull<RowT><<<dim3(nbh + nbl, npull), 256, 0, s>>>(gd, wd, ph, l, nbh, lo, hi, x + chunk * r, d->wc);
        L.check(__LINE__);
    }
    dist_allgather(L.g, x, chunk, s);
    const uint64_t total = (uint64_t)d->nranks * d->wc * 32;
    k_vp_apply<RowT><<<dim3((uint32_t)std::min<uint64_t>((total + 255) / 256, 148 * 8), npull), 256, 0, s>>>(
        gd, wd, ph, l, x, d->wc, d->nranks, d->d_bounds, npull);
    L.check(__LINE__);
}

// One vertex-partitioned PUSH level (default VP mode): every rank walks the
// out-edges of the frontier nodes it owns and ORs newly reachable cells into the owners' bit
// planes (peer memory in a real run: the fused exchange), then the planes are made visible
// to every rank and applied to the replicated H.  Per-rank edge work = the frontier's edges
// owned by the rank; no pass over all V.
template <class RowT>
void vp_level_push(Launch &L, const GraphDev &gd, const WsDev &wd, int ph, uint32_t l, uint32_t npull, bool wide) {
    DistState *d = L.g->dist;
    cudaStream_t s = L.s;
    dist_push_setup(L.g, wd.nslots);
    const size_t chunk = (size_t)npull * sizeof(RowT) * d->wc;
    const bool real = d->comm != nullptr && d->nranks > 1;
    uint32_t *const *xs = dist_push_targets(L.g);
    if (!real)  // the slices of this level start empty (a real run clears them in the exchange)
        CUDA_TRY(cudaMemset2DAsync(d->d_slices, d->slice_words * 4, 0, chunk * 4, d->nranks, s));
    for (int r = 0; r < d->nranks; r++) {
        if (!d->simulated && r != d->rank) continue;
        const VpPush vp{d->bounds[r], d->bounds[r + 1], (uint32_t)d->nranks, d->wc,
                        (uint32_t)(d->simulated ? r == 0 : 1), d->d_bounds, xs};
        if (wide)
            k_expand<RowT, true, true><<<148 * 8, 256, 0, s>>>(gd, wd, ph, l, vp);
        else
            k_expand<RowT, false, true><<<148 * 8, 256, 0, s>>>(gd, wd, ph, l, vp);
        L.check(__LINE__);
    }
    const VpPush vph{0, gd.V, (uint32_t)d->nranks, d->wc, 1, d->d_bounds, xs};
    k_expand_heavy<RowT, true><<<148 * 8, 256, 0, s>>>(gd, wd, ph, l, vph);
    L.check(__LINE__);
    size_t stride = 0;
    const uint32_t *x = dist_push_exchange(L.g, chunk, s, &stride);
    const uint32_t words = (uint32_t)d->nranks * d->wc;
    k_vp_apply_words<RowT><<<dim3(std::min<uint32_t>((words + 255) / 256, 148 * 8), npull), 256, 0, s>>>(
        gd, wd, ph, l, x, stride, d->wc, (uint32_t)d->nranks, d->d_bounds);
    L.check(__LINE__);
}

// Runs one exploration loop over all slots (lock-step).  For run 2 the per-level attach /
// RPG recovery / decide kernels run before the plan.  Returns when no slot expands.
template <class RowT, class RowC>
void run_phase(Launch &L, const GraphDev &gd, Workspace *ws, int ph, int hitting_mode, uint32_t max_levels,
               uint64_t total_cands) {
    cudaStream_t s = L.s;
    const bool vp = L.g->vp();  // vertex-partitioned: every level is a partitioned pull + all-gather
    const bool wide_forced = getenv("RIKI_FORCE_WIDE") != nullptr;  // tests: 64-bit item loop at any size
    const bool pull = L.g->pull_on || vp;
    ws->track_reached = L.g->pull_on ? 1 : 0;
    WsDev wd = ws->dev();
    k_phase_begin<<<(wd.nslots + 127) / 128, 128, 0, s>>>(wd, ph, hitting_mode);
    L.check(__LINE__);
    bool joint = false;
    if constexpr (sizeof(RowT) <= 4) joint = wd.hnode != 0;
    if (joint) {
        if constexpr (sizeof(RowT) <= 4) {
            k_fill_H_nodemajor<RowT><<<148 * 16, 256, 0, s>>>(wd, ph);
            L.check(__LINE__);
        }
        CUDA_TRY(cudaMemsetAsync(ws->ctr + C_JQN0, 0, 8, s));
    } else {
        k_fill_H<RowT><<<dim3(grid_of(ws->V, 256, 64), wd.nslots), 256, 0, s>>>(wd, ph);
        L.check(__LINE__);
    }
    k_seed<RowT><<<dim3(16, wd.nslots), 256, 0, s>>>(gd, wd, ph);
    L.check(__LINE__);
    // The host checks for termination only every LEVEL_BATCH levels: all per-level kernels
    // use fixed grids and read their work counts on the device, so levels past a slot's end
    // are device-side no-ops and the number of host synchronisations per run drops ~4x.
    static const bool trace_levels = getenv("RIKI_LEVELS") != nullptr;
    const bool no_graphs = getenv("RIKI_NO_GRAPHS") != nullptr || getenv("RIKI_SYNC") != nullptr;
    const bool wide = (uint64_t)wd.nslots * ws->qcap >= (1ull << 32) || wide_forced;
    // LEVEL_BATCH-level chunks replay as one CUDA graph (one launch instead of ~9 per level);
    // the per-level profiling events, the pull / vertex-partitioned levels (host-sized grids,
    // NCCL) and the level trace keep the plain launches
    const bool use_graphs = !no_graphs && !L.g->profiling && !pull && !joint && !trace_levels;
    // graph keys must not depend on the candidate count (a miss costs a capture and an
    // instantiation, milliseconds): grid-stride attach with one fixed grid
    // (sized by the slots in flight: a lone query's idle levels then cost a few blocks, not
    // 2368 -- single-query latency; full grids from 32 slots up)
    const uint32_t attach_blocks = total_cands ? std::min<uint32_t>(148 * 16, 64 * wd.nslots) : 0;
    const uint32_t rpg0_blocks = std::min<uint32_t>(148 * tier0_blocks_per_sm(k_extract_rpg<RowT, 0>), 32 * wd.nslots);
    const uint32_t rpg1_blocks = std::min<uint32_t>(148 * 3, 8 * wd.nslots);
    const uint32_t pull_min = vp ? 0u : !L.g->pull_on ? 0xFFFFFFFFu : std::max<uint32_t>(ws->V / PULL_MIN_DIV, 1);
    auto level_pre = [&](uint32_t l) {  // run 2: attach / RPG recovery / decide; then the plan
        if (ph == 1) {
            k_reset_level_ctrs<<<1, 1, 0, s>>>(wd);
            L.check(__LINE__);
            if (total_cands) {
                k_attach<RowT><<<attach_blocks, 256, 0, s>>>(wd);
                L.check(__LINE__);
                auto recover = [&]() {
                    k_extract_rpg<RowT, 0><<<rpg0_blocks, tier_threads<0>(), smem_ex<0>(), s>>>(gd, wd);
                    L.check(__LINE__);
                    k_extract_rpg<RowT, 1><<<rpg1_blocks, 256, smem_ex<1>(), s>>>(gd, wd);
                    L.check(__LINE__);
                    k_extract_rpg_big<RowT><<<ws->big_ctas, 256, 0, s>>>(gd, wd);
                    L.check(__LINE__);
                };
                if (wd.bounded) {  // two waves of bounded RPG recovery (k_rpg_select)
                    // RIKI_RPG_WAVES=1: a single flush wave (filter by the k-th key at the level start)
                    static const int waves = getenv("RIKI_RPG_WAVES") && atoi(getenv("RIKI_RPG_WAVES")) == 1 ? 1 : 2;
                    for (int wave = 2 - waves; wave < 2; wave++) {
                        k_reset_level_ctrs<<<1, 1, 0, s>>>(wd);
                        L.check(__LINE__);
                        k_rpg_select<<<wd.nslots, 256, U128_SORT_KEYS * 16, s>>>(wd, l, wave);
                        L.check(__LINE__);
                        recover();
                    }
                } else {
                    recover();
                }
            }
            k_decide_m<<<wd.nslots, 256, U128_SORT_KEYS * 16, s>>>(wd, l);
            L.check(__LINE__);
        }
        k_plan<<<1, MAX_SLOTS, 0, s>>>(wd, ph, l, pull_min);
        L.check(__LINE__);
    };
    auto level_expand = [&](uint32_t l) {
        if (joint) {
            if constexpr (sizeof(RowT) <= 4) {
                k_jexpand<RowT, false><<<148 * 8, 256, 0, s>>>(gd, wd, ph, l);
                L.check(__LINE__);
                k_jexpand<RowT, true><<<148 * 8, 256, 0, s>>>(gd, wd, ph, l);
                L.check(__LINE__);
            }
        } else {  // profiling: the variants that also count the relaxation atomics (CNT)
            // (a batch: with a few queries in flight L2 is not thrashed, and a lone query's flood
            // level wants every warp -- single-query p99 at config 5 was 71 ms at 4 blocks/SM)
            const bool big = ws->V >= EXP_BIG_V && wd.nslots >= 8 && !getenv("RIKI_NO_BIGOCC");
            if (L.g->profiling) {
                if (big) expand_launch<RowT, true, true>(L, gd, wd, ph, l, wide);
                else expand_launch<RowT, true, false>(L, gd, wd, ph, l, wide);
            } else {
                if (big) expand_launch<RowT, false, true>(L, gd, wd, ph, l, wide);
                else expand_launch<RowT, false, false>(L, gd, wd, ph, l, wide);
            }
        }
    };
    if (use_graphs && !getenv("RIKI_CHUNK_GRAPHS")) {
        // The whole run as ONE graph: a device-side while loop (conditional node) around one
        // level's kernels, the level index in ctr[C_LEVEL], the continue decision taken by
        // k_loop_cond from the plan's active-slot count -- no host round trip per level.
        struct Key {
            int ph;
            uint32_t max_levels, rbT, rbC, wide, attach_blocks, big_ctas, tier0, whole;
            WsDev wd;
            GraphDev gd;
        } key;
        memset(&key, 0, sizeof(key));
        key.ph = ph; key.max_levels = max_levels; key.rbT = sizeof(RowT); key.rbC = sizeof(RowC); key.wide = wide;
        key.attach_blocks = attach_blocks; key.big_ctas = ws->big_ctas; key.whole = 1;
        key.tier0 = tier0_blocks_per_sm(k_extract_rpg<RowT, 0>);
        key.wd = wd; key.gd = gd;
        const uint8_t *kb = (const uint8_t *)&key;
        Workspace::GraphEntry *hit = nullptr;
        for (Workspace::GraphEntry &e : ws->gcache)
            if (e.key.size() == sizeof(key) && !memcmp(e.key.data(), kb, sizeof(key))) { hit = &e; break; }
        if (!hit) {
            if (ws->gcache.size() >= 512) ws->clear_graphs();
            cudaGraph_t graph = nullptr;
            CUDA_TRY(cudaGraphCreate(&graph, 0));
            cudaGraphExec_t exec = nullptr;
            uint64_t before = L.launches;
            try {
                cudaGraphConditionalHandle h;
                CUDA_TRY(cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault));
                cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
                cp.conditional.handle = h;
                cp.conditional.type = cudaGraphCondTypeWhile;
                cp.conditional.size = 1;
                cudaGraphNode_t wn;
                CUDA_TRY(cudaGraphAddNode(&wn, graph, nullptr, 0, &cp));
                cudaGraph_t body = cp.conditional.phGraph_out[0];
                CUDA_TRY(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
                try {
                    level_pre(LV_DEVICE);
                    level_expand(LV_DEVICE);
                    k_loop_cond<<<1, 1, 0, s>>>(wd, h, max_levels);
                    L.check(__LINE__);
                } catch (...) {
                    cudaGraph_t dummy = nullptr;
                    cudaStreamEndCapture(s, &dummy);
                    throw;
                }
                CUDA_TRY(cudaStreamEndCapture(s, &body));
                const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
                if (e != cudaSuccess) RIKI_THROW(RIKI_ECUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
            } catch (...) {
                cudaGraphDestroy(graph);
                throw;
            }
            cudaGraphDestroy(graph);
            ws->gcache.push_back({std::vector<uint8_t>(kb, kb + sizeof(key)), exec, (uint32_t)(L.launches - before)});
            L.launches = before;
            hit = &ws->gcache.back();
        }
        CUDA_TRY(cudaMemsetAsync(ws->ctr + C_LEVEL, 0, 4, s));
        CUDA_TRY(cudaGraphLaunch(hit->exec, s));
        L.launches += hit->kernels;  // kernels per level (the level count is known on the device only)
        L.levels += 1;
    } else
    for (uint32_t l = 0; l <= max_levels; l++) {
        if (use_graphs) {  // levels [l, l + n) as one graph, then the host termination check
            const uint32_t n = std::min<uint32_t>(LEVEL_BATCH - l % LEVEL_BATCH, max_levels + 1 - l);
            struct Key {
                int ph;
                uint32_t l0, n, rbT, rbC, wide, attach_blocks, big_ctas, tier0;
                WsDev wd;
                GraphDev gd;
            } key;
            memset(&key, 0, sizeof(key));
            key.ph = ph; key.l0 = l; key.n = n; key.rbT = sizeof(RowT); key.rbC = sizeof(RowC); key.wide = wide;
            key.attach_blocks = attach_blocks; key.big_ctas = ws->big_ctas;
            key.tier0 = tier0_blocks_per_sm(k_extract_rpg<RowT, 0>);
            key.wd = wd; key.gd = gd;
            const uint8_t *kb = (const uint8_t *)&key;
            Workspace::GraphEntry *hit = nullptr;
            for (Workspace::GraphEntry &e : ws->gcache)
                if (e.key.size() == sizeof(key) && !memcmp(e.key.data(), kb, sizeof(key))) { hit = &e; break; }
            if (!hit) {
                if (ws->gcache.size() >= 512) ws->clear_graphs();
                const uint64_t before = L.launches;
                cudaGraph_t graph = nullptr;
                CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
                try {
                    for (uint32_t i = 0; i < n; i++) {
                        level_pre(l + i);
                        level_expand(l + i);
                    }
                } catch (...) {
                    cudaStreamEndCapture(s, &graph);
                    if (graph) cudaGraphDestroy(graph);
                    throw;
                }
                CUDA_TRY(cudaStreamEndCapture(s, &graph));
                cudaGraphExec_t exec = nullptr;
                const cudaError_t e = cudaGraphInstantiate(&exec, graph, 0);
                cudaGraphDestroy(graph);
                if (e != cudaSuccess) RIKI_THROW(RIKI_ECUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e));
                ws->gcache.push_back({std::vector<uint8_t>(kb, kb + sizeof(key)), exec, (uint32_t)(L.launches - before)});
                L.launches = before;
                hit = &ws->gcache.back();
            }
            CUDA_TRY(cudaGraphLaunch(hit->exec, s));
            L.launches += hit->kernels;
            CUDA_TRY(cudaMemcpyAsync(ws->h_ctr, ws->ctr, C_NCTR * 4, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            L.levels += n;
            if (ws->h_ctr[C_ACTIVE] == 0) break;  // (the last level's expansion was a device no-op)
            l += n - 1;
            continue;
        }
        Nvtx lv;
        {
            char nm[48];
            snprintf(nm, sizeof nm, "riki.run%d.level%u", ph + 1, l);
            lv.begin(nm);
        }
        level_pre(l);
        if (l % LEVEL_BATCH == LEVEL_BATCH - 1 || l == max_levels || pull) {
            CUDA_TRY(cudaMemcpyAsync(ws->h_ctr, ws->ctr, C_NCTR * 4, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            if (ws->h_ctr[C_ACTIVE] == 0) break;
        }
        L.levels++;
        if (L.g->profiling) CUDA_TRY(cudaEventRecord(ws->event(L.nev++), s));
        if (vp && L.g->dist->push) {
            if (uint32_t npull = ws->h_ctr[C_NPULL]) vp_level_push<RowT>(L, gd, wd, ph, l, npull, wide);
        } else {
            level_expand(l);
        }
        if (vp && !L.g->dist->push) {
            if (uint32_t npull = ws->h_ctr[C_NPULL]) vp_level<RowT>(L, gd, wd, ph, l, npull);
        } else if (vp) {
        } else if (L.g->pull_on) {
            if (uint32_t npull = ws->h_ctr[C_NPULL]) {
                uint32_t nbh = (gd.Vh + 7) / 8;
                uint32_t nbl = std::min<uint32_t>((ws->V - gd.Vh + 255) / 256, 148 * 8);
                k_pull<RowT><<<dim3(nbh + std::max<uint32_t>(nbl, 1), npull), 256, 0, s>>>(gd, wd, ph, l, nbh, 0u, ws->V,
                                                                                           nullptr, 0u);
                L.check(__LINE__);
            }
        }
        if (L.g->profiling) {  // events are read after the batch: no extra sync per level
            CUDA_TRY(cudaEventRecord(ws->event(L.nev++), s));
            L.expand_launches += 2 + (ws->h_ctr[C_NPULL] ? 1 : 0);
        }
        if (trace_levels) {  // diagnostics: per-level frontier / edge / new-cell counts (syncs every level)
            static unsigned long long last[P_NPROF];
            unsigned long long pr[P_NPROF];
            uint32_t c[C_NCTR];
            CUDA_TRY(cudaMemcpyAsync(c, ws->ctr, sizeof(c), cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaMemcpyAsync(pr, ws->prof, sizeof(pr), cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaStreamSynchronize(s));
            if (l == 0) memcpy(last, pr, sizeof(pr));
            fprintf(stderr, "[riki-level] ph=%d l=%u active=%u items=%u heavy_chunks=%u edges=%llu cells=%llu"
                            " dup=%llu blocked=%llu idle=%llu work=%llu\n", ph, l,
                    c[C_ACTIVE], c[C_TOTAL], c[C_NHEAVY], pr[P_EDGES] - last[P_EDGES], pr[P_NEWCELLS] - last[P_NEWCELLS],
                    pr[P_X_DUP] - last[P_X_DUP], pr[P_X_BLOCKED] - last[P_X_BLOCKED], pr[P_X_IDLE] - last[P_X_IDLE],
                    pr[P_X_WORK] - last[P_X_WORK]);
            memcpy(last, pr, sizeof(pr));
        }
    }
    if (joint) {
        k_jclear<<<64, 256, 0, s>>>(wd, 0);
        k_jclear<<<64, 256, 0, s>>>(wd, 1);
        L.check(__LINE__);
    }
}

template <class RowC, class RowM>
void run_batch_t(Launch &L, riki_graph *g, Workspace *ws, uint32_t depth) {
    cudaStream_t s = L.s;
    GraphDev gd = g->dev();
    WsDev wd = ws->dev();
    CUDA_TRY(cudaMemsetAsync(ws->arena_used, 0, 8, s));
    CUDA_TRY(cudaMemsetAsync(ws->out_used, 0, 8, s));
    CUDA_TRY(cudaMemsetAsync(ws->ctr, 0, C_NCTR * 4, s));
    {   // memo maps: clear only the keyword columns this batch can use (row words bound them)
        const size_t col = (size_t)MAPCAP * 16, pitch = 16 * col;
        CUDA_TRY(cudaMemset2DAsync(ws->mtab, pitch, 0xFF, sizeof(RowC) * col, wd.nslots, s));
        CUDA_TRY(cudaMemset2DAsync((uint8_t *)ws->mtab + 8 * col, pitch, 0xFF, sizeof(RowM) * col, wd.nslots, s));
    }
    // ---- run 1: central keywords
    Nvtx nv;
    nv.begin("riki.central_run");
    L.t0 = std::chrono::steady_clock::now();
    run_phase<RowC, RowC>(L, gd, ws, 0, -1, depth + 1, 0);
    L.mark(0);
    nv.begin("riki.cg_recovery");
    // ---- candidate CGs + recovery
    {   // (S^c, v) order of every slot's candidates: one segmented radix sort over the slots
        // (keys: level < 2^8 above a 32-bit caller id), then the candidate records
        const uint32_t G = ws->sort_group;
        k_cand_segments<<<(wd.nslots + 127) / 128, 128, 0, s>>>(wd, ws->seg_b, ws->seg_e, G);
        L.check(__LINE__);
        for (uint32_t s0 = 0; s0 < wd.nslots; s0 += G) {
            const uint32_t ng = std::min(G, wd.nslots - s0);
            size_t tb = ws->sort_tmp_bytes;
            CUDA_TRY(cub::DeviceSegmentedRadixSort::SortKeys(
                ws->sort_tmp, tb, (const unsigned long long *)ws->ck + (size_t)s0 * ws->capc,
                (unsigned long long *)ws->ck2 + (size_t)s0 * ws->capc, (int)((size_t)ng * ws->capc), (int)ng,
                ws->seg_b + s0, ws->seg_e + s0, 0, 40, s));
            L.launches += 2;
        }
        k_cand_sort<<<wd.nslots, 1024, 0, s>>>(gd, wd, ws->ck2);
        L.check(__LINE__);
    }
    k_scan_cands<<<1, MAX_SLOTS, 0, s>>>(wd);
    L.check(__LINE__);
    CUDA_TRY(cudaMemcpyAsync(ws->h_ctr, ws->ctr, C_NCTR * 4, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    uint64_t total_cands = ws->h_ctr[C_NCAND_TOTAL];
    if (total_cands) {
        k_extract_cg<RowC, 0><<<grid_of(total_cands, Tier<0>::GROUPS, 148 * tier0_blocks_per_sm(k_extract_cg<RowC, 0>)), tier_threads<0>(),
                                 smem_ex<0>(), s>>>(gd, wd);
        L.check(__LINE__);
        k_extract_cg<RowC, 1><<<148 * 3, 256, smem_ex<1>(), s>>>(gd, wd);
        L.check(__LINE__);
        k_extract_cg_big<RowC><<<ws->big_ctas, 256, 0, s>>>(gd, wd);
        L.check(__LINE__);
    }
    if (ws->beam_tie) {  // beam_mode 1 + tie-break (R29): truncate the recovered beam by W(CG)
        k_tie_weights<<<dim3(64, wd.nslots), 256, SORT_SMEM * 4, s>>>(gd, wd, true);
        L.check(__LINE__);
        k_beam_tie<<<wd.nslots, 256, U128_SORT_KEYS * 16, s>>>(wd);
        L.check(__LINE__);
        k_scan_cands<<<1, MAX_SLOTS, 0, s>>>(wd);
        L.check(__LINE__);
    }
    if (L.g->profiling) CUDA_TRY(cudaStreamSynchronize(s));
    L.mark(1);
    // ---- run 2: marginal keywords
    // Bounded recovery adds two selection waves (10 launches) per level and saves the RPG
    // recovery of candidates that cannot enter the top-k: it pays off when the candidate sets
    // are large against k (C5: ~300 k per query, +9 %; C2: ~47 k, -3 %: r02f A/B), hence the
    // crossover below.  RIKI_EAGER_RPG=1 / RIKI_BOUNDED_RPG=1 force either mode (A/B, tests).
    nv.begin("riki.marginal_run");
    const uint64_t per_slot = total_cands / std::max<uint32_t>(wd.nslots, 1);
    ws->bounded = getenv("RIKI_EAGER_RPG") ? 0 : getenv("RIKI_BOUNDED_RPG") ? 1 : per_slot > 100ull * ws->kmax;
    run_phase<RowM, RowC>(L, gd, ws, 1, -1, depth + 1, total_cands);
    L.mark(2);
    nv.begin("riki.finalize");
    // ---- top-k and packing
    k_final_select<<<wd.nslots, 256, U128_SORT_KEYS * 16, s>>>(wd);
    L.check(__LINE__);
    if (ws->tie_break) {  // R29 weight-sum tie-break
        k_tie_weights<<<dim3(64, wd.nslots), 256, SORT_SMEM * 4, s>>>(gd, wd, false);
        L.check(__LINE__);
        k_tie_select<<<wd.nslots, 256, U128_SORT_KEYS * 16, s>>>(wd);
        L.check(__LINE__);
    }
    k_final_lists<RowC><<<dim3(ws->kmax, wd.nslots), 256, SORT_SMEM * 4, s>>>(gd, wd);
    L.check(__LINE__);
    if (L.g->profiling) CUDA_TRY(cudaStreamSynchronize(s));
    L.mark(3);
}

template <class RowC>
void run_batch_c(Launch &L, riki_graph *g, Workspace *ws, uint32_t depth) {
    switch (ws->last_rb[1]) {
        case 2: run_batch_t<RowC, uint16_t>(L, g, ws, depth); break;
        case 4: run_batch_t<RowC, uint32_t>(L, g, ws, depth); break;
        default: run_batch_t<RowC, uint64_t>(L, g, ws, depth); break;
    }
}
void run_batch(Launch &L, riki_graph *g, Workspace *ws, uint32_t depth) {
    switch (ws->last_rb[0]) {
        case 2: run_batch_c<uint16_t>(L, g, ws, depth); break;
        case 4: run_batch_c<uint32_t>(L, g, ws, depth); break;
        default: run_batch_c<uint64_t>(L, g, ws, depth); break;
    }
}

// H layout of a batch: node-major (joint traversal) for large batches whose rows are <= 4
// bytes and whose padded slot rows fit one warp-wide 512-byte read; slot-major otherwise.
constexpr uint32_t JT_MIN_SLOTS = 32;
void set_layout(riki_graph *g, Workspace *ws, uint32_t n) {
    uint32_t rbmax = std::max(ws->last_rb[0], ws->last_rb[1]);
    uint32_t SP = (n + 7) & ~7u;
    ws->hnode = g->joint_on && rbmax <= 4 && n >= JT_MIN_SLOTS && SP * rbmax <= 512 ? 1 : 0;
    ws->SP = ws->hnode ? SP : 0;
}

// bytes per H row for T keywords: 2 (T <= 2), 4 (T <= 4) or 8
int row_bytes(uint32_t T) {
#ifdef RIKI_NO_U16
    return T <= 4 ? 4 : 8;
#else
    return T <= 2 ? 2 : (T <= 4 ? 4 : 8);
#endif
}

// qmap (optional): the batch runs in row-width groups; slot s takes query qmap[q0 + s]
// (positions q0 + s < nq of the grouped order), else query q0 + s.
__global__ void k_slots_from_device(SlotState *st, uint32_t nslots, uint32_t q0, uint32_t nq, const uint64_t *cptr,
                                    const uint32_t *ct, const uint64_t *mptr, const uint32_t *mt, SlotState tmpl,
                                    const uint64_t *tptr, uint32_t n_terms, const uint32_t *qmap) {
    uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= nslots) return;
    SlotState x = tmpl;
    x.active = q0 + s < nq;
    const uint32_t q = x.active && qmap ? qmap[q0 + s] : q0 + s;
    if (x.active) {
        uint64_t cb = cptr[q], ce = cptr[q + 1], mb = mptr[q], me = mptr[q + 1];
        x.T[0] = (uint32_t)(ce - cb);
        x.T[1] = (uint32_t)(me - mb);
        if (x.T[0] == 0 || x.T[0] > RIKI_MAX_TERMS || x.T[1] > RIKI_MAX_TERMS) x.err |= E_UNRESOLVED;
        for (uint32_t j = 0; j < x.T[0] && j < RIKI_MAX_TERMS; j++) x.term[0][j] = ct[cb + j];
        for (uint32_t j = 0; j < x.T[1] && j < RIKI_MAX_TERMS; j++) x.term[1][j] = mt[mb + j];
        for (int p = 0; p < 2; p++)
            for (uint32_t j = 0; j < x.T[p] && j < RIKI_MAX_TERMS; j++) {
                uint32_t t = x.term[p][j];
                if (t >= n_terms || tptr[t + 1] == tptr[t]) x.err |= E_UNRESOLVED;
            }
    } else {
        x.T[0] = x.T[1] = 0;
    }
    st[s] = x;
}

SlotState make_template(uint32_t k, uint32_t depth, const riki_params &p) {
    SlotState t;
    memset(&t, 0, sizeof(t));
    t.k = k;
    t.w = p.beam_w ? p.beam_w : k;
    t.depth = depth;
    t.beam_mode = p.beam_mode;
    t.tie_break = p.tie_break;
    t.ptc_mode = p.ptc_mode;
    t.early_term = p.early_term;
    t.gamma = p.gamma;
    t.L_end[0] = t.L_end[1] = -1;
    return t;
}

uint32_t auto_slots(riki_graph *g, uint32_t nq, uint32_t rb0, uint32_t rb1, uint32_t want_hint = 0) {
    uint32_t want = want_hint ? want_hint : g->batch_slots ? g->batch_slots : 256;
    want = std::min<uint32_t>(want, MAX_SLOTS);
    want = std::min<uint32_t>(want, std::max<uint32_t>(nq, 1));
    // an existing workspace that already fits needs no memory query (cudaMemGetInfo can take
    // tens of milliseconds)
    if (g->ws && g->ws->slots >= want && g->ws->hcap[0] >= rb0 && g->ws->hcap[1] >= rb1) return want;
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    uint64_t per = (uint64_t)g->V * (rb0 + rb1 + 8) + 16384ull * (8 + sizeof(Cand) + 16 + 8 + 8) +
                   16ull * 8192 * 16 + 64 * 1024;
    uint64_t budget = fr > (4ull << 30) ? (fr - (4ull << 30)) / 2 : fr / 4;
    uint32_t fit = (uint32_t)std::max<uint64_t>(1, budget / std::max<uint64_t>(per, 1));
    return std::max<uint32_t>(1, std::min(want, fit));
}

void collect_results(riki_graph *g, Workspace *ws, uint32_t n_active, const std::vector<uint32_t> &qidx,
                     std::vector<riki_results *> *out, cudaStream_t s) {
    const uint32_t ns = ws->cur ? ws->cur : ws->slots;
    if (n_active > ns || qidx.size() < n_active)
        RIKI_THROW(RIKI_EINVAL, "results of " + std::to_string(n_active) + " queries requested from a batch of " +
                                    std::to_string(ns) + " slots");
    std::vector<SlotState> st(ns);
    std::vector<OutHdr> hdr((size_t)ns * ws->kmax);
    unsigned long long used = 0;
    CUDA_TRY(cudaMemcpyAsync(st.data(), ws->st, st.size() * sizeof(SlotState), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(hdr.data(), ws->hdr, hdr.size() * sizeof(OutHdr), cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaMemcpyAsync(&used, ws->out_used, 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    std::vector<uint32_t> lists(used);
    if (used) CUDA_TRY(cudaMemcpyAsync(lists.data(), ws->out, used * 4, cudaMemcpyDeviceToHost, s));
    std::vector<uint64_t> cks;
    if (g->debug) {
        cks.resize((size_t)ns * ws->capc);
        CUDA_TRY(cudaMemcpyAsync(cks.data(), ws->ck, cks.size() * 8, cudaMemcpyDeviceToHost, s));
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    for (uint32_t sl = 0; sl < n_active; sl++) {
        const SlotState &x = st[sl];
        riki_results *r = new riki_results();
        r->nc = x.T[0];
        r->nm = x.T[1];
        r->stats.L_central = x.L_end[0];
        r->stats.L_marginal = x.T[1] ? x.L_end[1] : -1;
        r->stats.n_candidates = x.ncand_kept;
        r->stats.n_attached = x.n_attached;
        r->stats.n_ptc_fail = x.n_ptc_fail;
        r->stats.relax_central = x.relax[0];
        r->stats.relax_marginal = x.T[1] ? x.relax[1] : 0;
        for (uint32_t i = 0; i < x.nres; i++) {
            const OutHdr &h = hdr[(size_t)sl * ws->kmax + i];
            HostRPG p;
            p.central_node = h.central; p.sc = h.sc; p.sm = h.sm; p.score = h.score; p.ptc = (uint8_t)h.ptc;
            p.nodes.assign(lists.begin() + h.nodes_off, lists.begin() + h.nodes_off + h.n_nodes);
            p.vc.assign(lists.begin() + h.vc_off, lists.begin() + h.vc_off + h.n_vc);
            p.edges.assign(lists.begin() + h.edges_off, lists.begin() + h.edges_off + h.n_edges);
            memcpy(p.cdist, h.cdist, RIKI_MAX_TERMS);
            memcpy(p.mdist, h.mdist, RIKI_MAX_TERMS);
            r->rpgs.push_back(std::move(p));
        }
        if (g->debug) {
            uint32_t n = std::min(x.ncand_kept, ws->capc);
            r->cand.assign(cks.begin() + (size_t)sl * ws->capc, cks.begin() + (size_t)sl * ws->capc + n);
        }
        (*out)[qidx[sl]] = r;
    }
}

std::string err_text(uint32_t e) {
    std::string m;
    if (e & E_CAND) m += " candidate-capacity";
    if (e & E_HEAVY) m += " heavy-queue";
    if (e & E_ARENA) m += " arena";
    if (e & E_EXTRACT) m += " recovery-scratch";
    if (e & E_OUT) m += " output";
    if (e & E_UNRESOLVED) m += " unresolved-term";
    if (e & E_QUEUE) m += " frontier-queue";
    return m;
}

// Run [q0, q0+n) of a batch whose slot states are already on the device (any source).
// Grows capacities and re-runs when a workspace overflow is reported.
// Returns false when the batch needs more recovery arena than 32-bit offsets address: the
// caller re-runs it in smaller chunks (caps.slots halved).
// shape of a batch the remembered chunk size applies to (depth, row widths, k)
uint64_t slots_cap_key(const Caps &c, uint32_t depth) {
    return (uint64_t)depth << 40 | (uint64_t)c.rb[0] << 32 | (uint64_t)c.rb[1] << 24 | c.kmax;
}

bool run_with_retry(riki_graph *g, Launch &L, uint32_t depth, Caps &caps, uint32_t n_active,
                    const std::function<void()> &upload, std::vector<SlotState> *st_out) {
    for (int attempt = 0;; attempt++) {
        ensure_workspace(g, caps);
        Workspace *ws = g->ws;
        upload();
        run_batch(L, g, ws, depth);
        const uint32_t ns = ws->cur ? ws->cur : ws->slots;
        st_out->resize(ns);
        CUDA_TRY(cudaMemcpyAsync(st_out->data(), ws->st, ns * sizeof(SlotState), cudaMemcpyDeviceToHost, L.s));
        CUDA_TRY(cudaStreamSynchronize(L.s));
        uint32_t err = 0;
        for (uint32_t i = 0; i < n_active; i++) err |= (*st_out)[i].err;
        if (err & E_UNRESOLVED) RIKI_THROW(RIKI_EUNRESOLVED, "a query term is unresolved (empty posting) or out of range");
        if (!err) return true;
        g->stats.retries++;
        if (getenv("RIKI_TRACE")) fprintf(stderr, "[riki] retry after overflow:%s\n", err_text(err).c_str());
        if (attempt >= 6) RIKI_THROW(RIKI_ENOMEM, "workspace overflow:" + err_text(err));
        if (err & E_CAND) caps.capc = std::min<uint32_t>(caps.capc * 4, next_pow2(g->V + 1));
        if (err & (E_ARENA | E_EXTRACT)) {
            // arena offsets are 32-bit words (EMPTY = 0xFFFFFFFF is the failure sentinel)
            const uint64_t amax = g->arena_limit ? std::min<uint64_t>(g->arena_limit, ARENA_MAX_WORDS) : ARENA_MAX_WORDS;
            if (caps.arena >= amax) {
                if (n_active <= 1) RIKI_THROW(RIKI_ENOMEM, "recovery arena exceeds 2^32 words for one query");
                const bool full_chunk = n_active >= caps.slots;  // not a short tail chunk
                caps.slots = std::max(1u, n_active / 2);
                if (full_chunk) {  // remembered for later batches of the same shape only
                    g->slots_cap = caps.slots;
                    g->slots_cap_key = slots_cap_key(caps, depth);
                }
                return false;
            }
            caps.arena = std::min<uint64_t>(caps.arena * 4, amax);
        }
        if (err & E_OUT) caps.out *= 4;
        if (err & E_QUEUE) caps.qcap = 2 * g->V;  // exact bound: one retained + one new entry per node
        if (err & E_HEAVY) RIKI_THROW(RIKI_ENOMEM, "heavy work queue overflow");
    }
}

void add_stats(riki_graph *g, Workspace *ws, Launch &L, uint32_t nq) {
    unsigned long long prof[P_NPROF];
    CUDA_TRY(cudaMemcpyAsync(prof, ws->prof, sizeof(prof), cudaMemcpyDeviceToHost, L.s));
    CUDA_TRY(cudaStreamSynchronize(L.s));
    for (uint32_t i = 0; i + 1 < L.nev; i += 2) {
        float ms = 0;
        CUDA_TRY(cudaEventElapsedTime(&ms, ws->event(i), ws->event(i + 1)));
        L.expand_ms += ms;
    }
    L.nev = 0;
#if REC_STATS
    fprintf(stderr, "[riki-rec] builds %llu edges %llu max %llu build_cyc %llu | waits %llu wait_cyc %llu | items %llu | "
                    "cg cands %llu cand_cyc %llu cand_max %llu warp_max %llu hist %llu %llu %llu %llu %llu %llu\n",
            prof[P_R_BUILDS], prof[P_R_BEDGES], prof[P_R_BMAX], prof[P_R_BCYC], prof[P_R_WAITS], prof[P_R_WCYC],
            prof[P_R_ITEMS], prof[P_R_CANDS], prof[P_R_CANDCYC], prof[P_R_CANDMAX], prof[P_R_WARPMAX],
            prof[P_R_H0], prof[P_R_H0 + 1], prof[P_R_H0 + 2], prof[P_R_H0 + 3], prof[P_R_H0 + 4], prof[P_R_H0 + 5]);
    fprintf(stderr, "[riki-rec] tiers: cg t1 %llu big %llu | rpg t1 %llu big %llu (nodes %llu edges %llu max edges %llu)\n",
            prof[P_R_T1], prof[P_R_T2], prof[P_R_T1RPG], prof[P_R_T2RPG], prof[P_R_T2NODES], prof[P_R_T2EDGES],
            prof[P_R_T2MAXE]);
#endif
    uint64_t rb = ws->last_rb[0];  // bytes per H row (approximation when phases differ)
    g->stats.expand_launches += L.expand_launches;
    g->stats.expand_ms += L.expand_ms;
    g->stats.expand_bytes += prof[P_ITEMS] * (12 + rb) + prof[P_EDGES] * (5 + rb) + prof[P_NEWCELLS] + prof[P_ENQ] * 4 +
                             prof[P_PULLNODES] * (8 + rb) + prof[P_PULLEDGES] * (5 + rb);
    g->stats.kernel_launches += L.launches;
    g->stats.queries += nq;
    g->stats.exp_items += prof[P_ITEMS];
    g->stats.exp_items_work += prof[P_ITEMS_WORK];
    g->stats.exp_edges += prof[P_EDGES] + prof[P_PULLEDGES];
    g->stats.exp_new_cells += prof[P_NEWCELLS];
    g->stats.exp_atomics += prof[P_ATOMS];
    g->stats.exp_enqueued += prof[P_ENQ];
    for (int i = 0; i < 4; i++) g->stats.section_ms[i] += L.sec_ms[i];
    g->stats.levels += L.levels;
    L.sec_ms[0] = L.sec_ms[1] = L.sec_ms[2] = L.sec_ms[3] = 0;
    L.levels = 0;
    L.launches = 0;
    L.expand_ms = 0;
    L.expand_launches = 0;
}

}  // namespace

static void check_query_host(riki_graph *g, const QueryIn &q) {
    if (q.nc == 0) RIKI_THROW(RIKI_EEMPTY_CENTRAL, "C must be non-empty (Def. RPQ, P:105)");
    if (q.nc > RIKI_MAX_TERMS || q.nm > RIKI_MAX_TERMS) RIKI_THROW(RIKI_EINVAL, "at most 8 terms per keyword class");
    for (uint32_t j = 0; j < q.nc + q.nm; j++) {
        uint32_t t = j < q.nc ? q.c[j] : q.m[j - q.nc];
        if (t >= g->n_terms) RIKI_THROW(RIKI_EINVAL, "term id " + std::to_string(t) + " out of range");
        if (g->h_tptr[t + 1] == g->h_tptr[t])
            RIKI_THROW(RIKI_EUNRESOLVED, "term " + std::to_string(t) + " (query position " + std::to_string(j) +
                                             ") has an empty posting list");
    }
}

static void check_common(riki_graph *g, uint32_t k, uint32_t depth, const riki_params &p) {
    if (!g->has_act) RIKI_THROW(RIKI_ENOWEIGHTS, "activation levels not set (call riki_set_*_weights)");
    if (k == 0) RIKI_THROW(RIKI_EINVAL, "k must be >= 1");
    if (depth > RIKI_MAX_DEPTH) RIKI_THROW(RIKI_EDEPTH, "depth must be <= 254");
    if (!(p.gamma >= 0.0 && p.gamma <= 1.0)) RIKI_THROW(RIKI_EINVAL, "gamma must be in [0,1]");
    if (p.beam_mode < 0 || p.beam_mode > 1) RIKI_THROW(RIKI_EINVAL, "beam_mode must be 0 or 1");
    if (p.tie_break != 0 && p.tie_break != 1) RIKI_THROW(RIKI_EINVAL, "tie_break must be 0 or 1");
    if (p.tie_break == 1 && !g->d_wfix)
        RIKI_THROW(RIKI_ENOWEIGHTS, "tie_break 1 needs the fine edge weights (set_edge/node/label_weights)");
    if (p.ptc_mode < 0 || p.ptc_mode > 3) RIKI_THROW(RIKI_EINVAL, "ptc_mode must be 0..3");
    if (p.early_term < 0 || p.early_term > 2) RIKI_THROW(RIKI_EINVAL, "early_term must be 0..2");
    if (p.beam_w && p.beam_w < k) RIKI_THROW(RIKI_EINVAL, "beam width must be >= k (P:309)");
}

static Caps initial_caps(riki_graph *g, uint32_t nq, uint32_t k, uint32_t rb0, uint32_t rb1, uint32_t depth,
                         uint32_t want_hint = 0) {
    Caps c;
    c.rb[0] = rb0;
    c.rb[1] = rb1;
    c.slots = auto_slots(g, nq, rb0, rb1, want_hint);
    c.capc = std::min<uint32_t>(16384, next_pow2(g->V + 1));
    c.kmax = std::max<uint32_t>(k, g->ws ? g->ws->kmax : 1);
    // a full-width batch of this shape overflowed the arena before: start at its chunk size
    if (g->slots_cap && g->slots_cap_key == slots_cap_key(c, depth)) c.slots = std::min(c.slots, g->slots_cap);
    c.arena = std::max<uint64_t>(64ull << 20, g->ws ? g->ws->arena_cap : 0);
    if (g->arena_limit) c.arena = std::min<uint64_t>(c.arena, g->arena_limit);
    c.out = std::max<uint64_t>(16ull << 20, g->ws ? g->ws->out_cap : 0);
    if (g->ws) c.capc = std::max(c.capc, g->ws->capc);
    c.qcap = std::max<uint32_t>(g->V, g->ws ? g->ws->qcap : 0);
    return c;
}

void engine_search(riki_graph *g, const std::vector<QueryIn> &qs, uint32_t k, uint32_t depth, const riki_params &p,
                   cudaStream_t stream, std::vector<riki_results *> *out) {
    check_common(g, k, depth, p);
    for (const QueryIn &q : qs) check_query_host(g, q);
    out->assign(qs.size(), nullptr);
    if (qs.empty()) return;
    Tracer tr;
    uint32_t maxc0 = 0, maxm0 = 0;
    for (const QueryIn &q : qs) { maxc0 = std::max(maxc0, q.nc); maxm0 = std::max(maxm0, q.nm); }
    Caps caps = initial_caps(g, (uint32_t)qs.size(), k, row_bytes(maxc0), row_bytes(std::max(maxm0, 1u)), depth);
    tr("initial_caps");
    // every launch and copy of the search is issued on the caller's stream when one is given
    // (ordered after the caller's earlier work on it), else on the library stream
    Launch L{g, stream ? stream : g->stream};
    if (g->ws) g->ws->last_n = 0;  // the workspace is reused: a pending device batch is gone
    for (riki_results *r : g->dev_stash) delete r;
    g->dev_stash.clear();
    SlotState tmpl = make_template(k, depth, p);
    std::vector<riki_results *> &res = *out;
    // row-width groups (see engine_search_device)
    auto cls_of = [&](uint32_t q) {
        return (uint32_t)row_bytes(std::max(qs[q].nc, 1u)) << 8 | (uint32_t)row_bytes(std::max(qs[q].nm, 1u));
    };
    const uint32_t nq = (uint32_t)qs.size();
    std::vector<uint32_t> order(nq);
    for (uint32_t q = 0; q < nq; q++) order[q] = q;
    if (!getenv("RIKI_NO_ROW_GROUPS"))
        std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return cls_of(a) < cls_of(b); });
    try {
        for (uint32_t q0 = 0; q0 < nq;) {
            ensure_workspace(g, caps);
            uint32_t slots = std::min(g->ws->slots, caps.slots);
            // a chunk never mixes row widths (RIKI_NO_ROW_GROUPS: one group at the widest rows)
            uint32_t n = std::min<uint32_t>(slots, nq - q0);
            if (!getenv("RIKI_NO_ROW_GROUPS"))
                for (uint32_t i = 1; i < n; i++)
                    if (cls_of(order[q0 + i]) != cls_of(order[q0])) { n = i; break; }
            uint32_t maxc = 0, maxm = 0;
            for (uint32_t i = 0; i < n; i++) {
                maxc = std::max(maxc, qs[order[q0 + i]].nc);
                maxm = std::max(maxm, qs[order[q0 + i]].nm);
            }
            std::vector<uint32_t> qidx(n);
            for (uint32_t i = 0; i < n; i++) qidx[i] = order[q0 + i];
            std::vector<SlotState> stv;
            auto upload = [&]() {
                Workspace *ws = g->ws;
                ws->last_rb[0] = row_bytes(maxc);
                ws->last_rb[1] = row_bytes(std::max(maxm, 1u));
                ws->tie_break = tmpl.tie_break;
                ws->beam_tie = tmpl.tie_break && tmpl.beam_mode == 1;
                ws->cur = n;
                set_layout(g, ws, n);
                std::vector<SlotState> h(n, tmpl);
                for (uint32_t i = 0; i < n; i++) {
                    SlotState &x = h[i];
                    const QueryIn &q = qs[qidx[i]];
                    x.active = 1;
                    x.T[0] = q.nc; x.T[1] = q.nm;
                    for (uint32_t j = 0; j < q.nc; j++) x.term[0][j] = q.c[j];
                    for (uint32_t j = 0; j < q.nm; j++) x.term[1][j] = q.m[j];
                }
                CUDA_TRY(cudaMemcpyAsync(ws->st, h.data(), h.size() * sizeof(SlotState), cudaMemcpyHostToDevice, L.s));
                CUDA_TRY(cudaMemsetAsync(ws->prof, 0, P_NPROF * 8, L.s));
            };
            tr("before run");
            if (!run_with_retry(g, L, depth, caps, n, upload, &stv)) continue;  // smaller chunk
            tr("run_with_retry");
            collect_results(g, g->ws, n, qidx, &res, L.s);
            tr("collect_results");
            add_stats(g, g->ws, L, n);
            tr("add_stats");
            q0 += n;
        }
    } catch (...) {
        for (auto *r : res) delete r;
        res.assign(qs.size(), nullptr);
        throw;
    }
}

void engine_search_device(riki_graph *g, uint32_t nq, const uint64_t *d_cptr, const uint32_t *d_cterms,
                          const uint64_t *d_mptr, const uint32_t *d_mterms, uint32_t k, uint32_t depth,
                          const riki_params &p) {
    check_common(g, k, depth, p);
    Tracer tr;
    // row widths need the max term counts: read the (small) pointer arrays' extents on device
    std::vector<uint64_t> cp(nq + 1), mp(nq + 1);
    CUDA_TRY(cudaMemcpyAsync(cp.data(), d_cptr, (nq + 1) * 8, cudaMemcpyDeviceToHost, g->stream));
    CUDA_TRY(cudaMemcpyAsync(mp.data(), d_mptr, (nq + 1) * 8, cudaMemcpyDeviceToHost, g->stream));
    CUDA_TRY(cudaStreamSynchronize(g->stream));
    uint32_t maxc = 0, maxm = 0;
    for (uint32_t q = 0; q < nq; q++) {
        maxc = std::max<uint32_t>(maxc, (uint32_t)(cp[q + 1] - cp[q]));
        maxm = std::max<uint32_t>(maxm, (uint32_t)(mp[q + 1] - mp[q]));
    }
    if (maxc > RIKI_MAX_TERMS || maxm > RIKI_MAX_TERMS) RIKI_THROW(RIKI_EINVAL, "at most 8 terms per keyword class");
    tr("ptr D2H");
    // Row-width groups: a lock-step batch uses one H row width per run (the widest query's),
    // so a mixed batch (config 5: |M| = 2 / 4 / 6) runs as one sub-batch per (central, marginal)
    // row width -- narrower rows for most queries: half the H bytes per relaxation and per
    // reset, and fewer registers in the expansion.  Results are per query either way.
    auto cls_of = [&](uint32_t q) {
        return (uint32_t)row_bytes(std::max<uint32_t>((uint32_t)(cp[q + 1] - cp[q]), 1u)) << 8 |
               (uint32_t)row_bytes(std::max<uint32_t>((uint32_t)(mp[q + 1] - mp[q]), 1u));
    };
    std::vector<uint32_t> order(nq);
    for (uint32_t q = 0; q < nq; q++) order[q] = q;
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return cls_of(a) < cls_of(b); });
    std::vector<std::pair<uint32_t, uint32_t>> groups;  // [begin, end) in `order`
    for (uint32_t i = 0; i < nq;) {
        uint32_t j = i + 1;
        while (j < nq && cls_of(order[j]) == cls_of(order[i])) j++;
        groups.push_back({i, j});
        i = j;
    }
    if (getenv("RIKI_NO_ROW_GROUPS")) {  // A/B: one group at the widest rows
        groups.assign(1, {0u, nq});
        for (uint32_t q = 0; q < nq; q++) order[q] = q;
    }
    const bool grouped = groups.size() > 1;
    if (grouped) {
        if (g->qmap_cap < nq) {
            if (g->d_qmap) cudaFree(g->d_qmap);
            g->d_qmap = nullptr;
            g->qmap_cap = 0;
            CUDA_TRY(cudaMalloc(&g->d_qmap, (size_t)nq * 4));
            g->qmap_cap = nq;
        }
        CUDA_TRY(cudaMemcpyAsync(g->d_qmap, order.data(), (size_t)nq * 4, cudaMemcpyHostToDevice, g->stream));
    }
    // the whole batch in flight when it fits the device memory (auto_slots), else chunks; the
    // workspace is sized for the widest rows, each group uses its own width inside it
    Caps caps = initial_caps(g, nq, k, row_bytes(std::max(maxc, 1u)), row_bytes(std::max(maxm, 1u)), depth,
                             std::max(g->batch_slots, std::min<uint32_t>(nq, MAX_SLOTS)));
    tr("initial_caps");
    ensure_workspace(g, caps);
    Launch L{g, g->stream};
    SlotState tmpl = make_template(k, depth, p);
    if (maxc == 0) RIKI_THROW(RIKI_EEMPTY_CENTRAL, "C must be non-empty (Def. RPQ, P:105)");
    std::vector<SlotState> stv;
    for (riki_results *r : g->dev_stash) delete r;
    g->dev_stash.clear();
    bool chunked = grouped;
    for (const auto &grp : groups) {
        const uint32_t gc = grouped ? cls_of(order[grp.first]) >> 8 : row_bytes(std::max(maxc, 1u));
        const uint32_t gm = grouped ? cls_of(order[grp.first]) & 0xFF : row_bytes(std::max(maxm, 1u));
        for (uint32_t q0 = grp.first; q0 < grp.second;) {
            const uint32_t n = std::min<uint32_t>(std::min(caps.slots, g->ws->slots), grp.second - q0);
            auto upload = [&]() {
                Workspace *ws = g->ws;
                ws->last_rb[0] = gc;
                ws->last_rb[1] = gm;
                ws->tie_break = tmpl.tie_break;
                ws->beam_tie = tmpl.tie_break && tmpl.beam_mode == 1;
                ws->cur = n;
                set_layout(g, ws, n);
                k_slots_from_device<<<(n + 127) / 128, 128, 0, L.s>>>(ws->st, n, q0, grp.second, d_cptr, d_cterms, d_mptr,
                                                                      d_mterms, tmpl, g->d_tptr, g->n_terms,
                                                                      grouped ? g->d_qmap : nullptr);
                L.check(__LINE__);
                CUDA_TRY(cudaMemsetAsync(ws->prof, 0, P_NPROF * 8, L.s));
            };
            tr("ensure+setup");
            if (!run_with_retry(g, L, depth, caps, n, upload, &stv)) {  // arena limit: smaller chunks
                chunked = true;
                continue;
            }
            tr("run_with_retry");
            if (chunked || n < nq) {  // results of a chunk leave HBM before the next chunk runs
                chunked = true;
                g->dev_stash.resize(nq, nullptr);
                std::vector<uint32_t> qidx(n);
                for (uint32_t i = 0; i < n; i++) qidx[i] = order[q0 + i];
                collect_results(g, g->ws, n, qidx, &g->dev_stash, L.s);
            }
            add_stats(g, g->ws, L, n);
            q0 += n;
        }
    }
    g->ws->last_n = nq;
    tr("add_stats");
}

void engine_fetch(riki_graph *g, uint32_t nq, std::vector<riki_results *> *out) {
    if (!g->ws || g->ws->last_n != nq) RIKI_THROW(RIKI_EINVAL, "no device batch of that size to fetch");
    if (!g->dev_stash.empty()) {  // the batch ran in chunks: results were collected per chunk
        *out = std::move(g->dev_stash);
        g->dev_stash.clear();
        g->ws->last_n = 0;
        return;
    }
    out->assign(nq, nullptr);
    std::vector<uint32_t> qidx(nq);
    for (uint32_t i = 0; i < nq; i++) qidx[i] = i;
    collect_results(g, g->ws, nq, qidx, out, g->stream);
    g->ws->last_n = 0;  // fetched once: a second fetch is an error, not a stale read
}

void engine_hitting_levels(riki_graph *g, const uint32_t *terms, uint32_t T, uint32_t depth, int block_mode,
                           uint8_t *H_out, uint8_t *block_out, uint64_t *relax_out, int32_t *L_out) {
    if (!g->has_act) RIKI_THROW(RIKI_ENOWEIGHTS, "activation levels not set");
    if (T == 0 || T > RIKI_MAX_TERMS) RIKI_THROW(RIKI_EINVAL, "1..8 terms");
    if (depth > RIKI_MAX_DEPTH) RIKI_THROW(RIKI_EDEPTH, "depth must be <= 254");
    if (block_mode < 0 || block_mode > 2) RIKI_THROW(RIKI_EINVAL, "block_mode must be 0, 1 or 2");
    if (!H_out || !block_out) RIKI_THROW(RIKI_EINVAL, "null output");
    QueryIn q{};
    q.nc = T;
    for (uint32_t j = 0; j < T; j++) q.c[j] = terms[j];
    check_query_host(g, q);
    Caps caps = initial_caps(g, 1, 1, row_bytes(T), 2, depth);
    if (g->ws) g->ws->last_n = 0;  // the workspace is reused: a pending device batch is gone
    for (riki_results *r : g->dev_stash) delete r;
    g->dev_stash.clear();
    for (int attempt = 0;; attempt++) {  // grows the frontier queues on E_QUEUE (see run_with_retry)
    ensure_workspace(g, caps);
    Workspace *ws = g->ws;
    ws->last_rb[0] = row_bytes(T);
    ws->last_rb[1] = 4;
    ws->hnode = 0;
    SlotState x = make_template(1, depth, riki_params{0.5, 0, 0, 0, 0, 0});
    x.w = 0xFFFFFFFFu;
    ws->cur = 1;
    std::vector<SlotState> h(1, x);
    h[0].active = 1;
    h[0].T[0] = T;
    for (uint32_t j = 0; j < T; j++) h[0].term[0][j] = terms[j];
    Launch L{g, g->stream};
    CUDA_TRY(cudaMemcpyAsync(ws->st, h.data(), h.size() * sizeof(SlotState), cudaMemcpyHostToDevice, L.s));
    CUDA_TRY(cudaMemsetAsync(ws->ctr, 0, C_NCTR * 4, L.s));
    CUDA_TRY(cudaMemsetAsync(ws->prof, 0, P_NPROF * 8, L.s));
    GraphDev gd = g->dev();
    uint8_t *dH = nullptr, *dB = nullptr;
    CUDA_TRY(cudaMalloc(&dH, (size_t)g->V * T + 1));
    CUDA_TRY(cudaMalloc(&dB, (size_t)g->V + 1));
    int blocking = block_mode == 1 || (block_mode == 2 && T >= 2);
    try {
        WsDev wd = ws->dev();
        if (ws->last_rb[0] == 2) {
            run_phase<uint16_t, uint16_t>(L, gd, ws, 0, block_mode, depth + 1, 0);
            k_pack_H<uint16_t><<<grid_of(g->V, 256), 256, 0, L.s>>>(gd, wd, T, dH, dB, blocking);
        } else if (T <= 4) {
            run_phase<uint32_t, uint32_t>(L, gd, ws, 0, block_mode, depth + 1, 0);
            k_pack_H<uint32_t><<<grid_of(g->V, 256), 256, 0, L.s>>>(gd, wd, T, dH, dB, blocking);
        } else {
            run_phase<uint64_t, uint64_t>(L, gd, ws, 0, block_mode, depth + 1, 0);
            k_pack_H<uint64_t><<<grid_of(g->V, 256), 256, 0, L.s>>>(gd, wd, T, dH, dB, blocking);
        }
        L.check(__LINE__);
        CUDA_TRY(cudaMemcpyAsync(H_out, dH, (size_t)g->V * T, cudaMemcpyDeviceToHost, L.s));
        CUDA_TRY(cudaMemcpyAsync(block_out, dB, g->V, cudaMemcpyDeviceToHost, L.s));
        SlotState s0;
        CUDA_TRY(cudaMemcpyAsync(&s0, ws->st, sizeof(SlotState), cudaMemcpyDeviceToHost, L.s));
        CUDA_TRY(cudaStreamSynchronize(L.s));
        if ((s0.err & E_QUEUE) && caps.qcap < 2 * g->V && attempt < 2) {
            caps.qcap = 2 * g->V;
            g->stats.retries++;
            cudaFree(dH);
            cudaFree(dB);
            continue;
        }
        if (s0.err) RIKI_THROW(RIKI_ENOMEM, "workspace overflow:" + err_text(s0.err));
        if (relax_out) *relax_out = s0.relax[0];
        if (L_out) *L_out = s0.L_end[0];
        add_stats(g, ws, L, 0);
    } catch (...) {
        cudaFree(dH);
        cudaFree(dB);
        throw;
    }
    cudaFree(dH);
    cudaFree(dB);
    return;
    }
}

void engine_free(riki_graph *g) {
    for (riki_results *r : g->dev_stash) delete r;
    g->dev_stash.clear();
    if (g->d_qmap) cudaFree(g->d_qmap);
    g->d_qmap = nullptr;
    g->qmap_cap = 0;
    if (g->ws) {
        g->ws->release();
        delete g->ws;
        g->ws = nullptr;
    }
}

uint64_t engine_workspace_bytes(const riki_graph *g) { return g->ws ? g->ws->bytes : 0; }
