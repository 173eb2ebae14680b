// gx_explore.cu -- level-synchronous BFS on the B200 (reference:
// explore.py:147-395, network.py:184-238), the per-level primitives of the
// hash-owner sharded multi-GPU driver, and the isolated FINDORPUT
// benchmark (bench.py:120-202 protocol).
#include <algorithm>
#include <cstring>
#include <vector>

#include "gx_expand.cuh"
#include "gx_staged.cuh"
#include "gx_internal.h"

#include "gx_level.cuh"
#include "gx_bench.cuh"

namespace gx {

// One BFS level.  Every warp takes 32 frontier states at a time:
//   count pass   successors and transitions per state (expand_state),
//                warp scan -> each lane's slice of the warp's successor list
//   emit pass    successors into the warp's shared-memory queue, QWORDS/V
//                at a time
//   filter       (V <= 2) drop successors the block-local cache has seen
//   probe        FINDORPUT of the queue: G lanes per key, U keys per lane
//                group with all first-bucket loads issued up front
//   stage        INSERTED keys go to a shared-memory out-queue, flushed to
//                the next frontier with one atomic per chunk
#ifndef GX_LEVEL_MINB
#define GX_LEVEL_MINB 2  // resident blocks per SM the level kernel is compiled for
#endif

template <int BW, int V, int G, bool MARK>
__global__ void __launch_bounds__(256, GX_LEVEL_MINB) k_level(TableDesc T, NetDesc N, LevelArgs A) {
    constexpr int QCAP = QWORDS_REG / V;
    __shared__ __align__(16) uint32_t qbuf[8][QWORDS_REG];
    __shared__ __align__(16) uint32_t obuf[8][QWORDS_REG];
    extern __shared__ unsigned long long dcache[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    constexpr bool CACHE_OK = MARK && V <= 2;
    const uint32_t cmask = CACHE_OK ? A.cache_mask : 0u;
    if (cmask) {
        for (uint32_t i = threadIdx.x; i <= cmask; i += blockDim.x) dcache[i] = 0ull;
        __syncthreads();
    }
    uint32_t* q = qbuf[wid];
    uint32_t* outq = obuf[wid];
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    const bool leader = MARK ? (lane & (G - 1)) == 0 : true;
    unsigned long long trans = 0, expanded = 0, probes = 0;
    for (uint64_t base = warp * 32; base < A.nfront; base += nwarps * 32) {
        int stop = 0;
        if (lane == 0)
            stop = (*(volatile unsigned long long*)&A.ctr[LV_FULL] != 0ull) ||
                   (*(volatile unsigned long long*)&A.ctr[LV_OVF] != 0ull);
        if (__shfl_sync(FULLMASK, stop, 0)) break;
        const uint64_t idx = base + lane;
        const bool has = idx < A.nfront;
        uint32_t s[V];
        if (has)
            load_state<V>(A.front + idx * V, s);
        else
#pragma unroll
            for (int w = 0; w < V; w++) s[w] = 0;
        uint64_t cnt = 0;
        uint32_t n = 0;
        if (has) {
            n = expand_state<V, false>(N, s, &cnt, 0, 0, nullptr);
            trans += cnt;
            expanded += 1;
            if (cnt == 0 && A.detect) {
                unsigned long long p = atomicAdd(&A.ctr[LV_DL], 1ull) - A.dl_base;
                if (p < A.dl_cap) store_state<V>(A.dl + p * V, s);
            }
        }
        uint32_t incl = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(FULLMASK, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t total = __shfl_sync(FULLMASK, incl, 31);
        const uint32_t excl = incl - n;
        for (uint32_t c0 = 0; c0 < total; c0 += QCAP) {
            const uint32_t c1 = min(total, c0 + (uint32_t)QCAP);
            if (has && n && excl < c1 && excl + n > c0) {
                const uint32_t lo = max(c0, excl) - excl;
                const uint32_t hi = min(c1, excl + n) - excl;
                uint64_t dummy;
                expand_state<V, true>(N, s, &dummy, lo, hi, q + (uint64_t)(excl + lo - c0) * V);
            }
            __syncwarp();
            uint32_t m = c1 - c0;
            if (CACHE_OK && cmask) m = cache_filter<V>(T, dcache, cmask, q, m);
            probes += lane == 0 ? m : 0;
            uint32_t n_out = 0;
            bool any_full = false;
            if constexpr (MARK) {
                using S = ProbeShape<BW, G>;
                for (uint32_t r0 = 0; r0 < m; r0 += S::KB) {
                    uint32_t own_key[S::M][V];
                    bool own_act[S::M];
#pragma unroll
                    for (int mm = 0; mm < S::M; mm++) {
                        const uint32_t e = r0 + lane + 32 * mm;
                        own_act[mm] = e < m;
#pragma unroll
                        for (int w = 0; w < V; w++) own_key[mm][w] = own_act[mm] ? q[e * V + w] : 0u;
                    }
                    uint32_t key[S::U][V];
                    bool act[S::U];
                    int code[S::U];
                    int64_t hd[S::U];
                    probe_batch<BW, V, G>(T, own_key, own_act, key, act, code, hd);
#pragma unroll
                    for (int u = 0; u < S::U; u++) {
                        const bool ins = leader && act[u] && code[u] == INSERTED;
                        any_full |= leader && act[u] && code[u] == TABLE_FULL;
                        const uint32_t insm = __ballot_sync(FULLMASK, ins);
                        if (ins) {
                            const uint32_t p = n_out + __popc(insm & lanemask_lt());
#pragma unroll
                            for (int w = 0; w < V; w++) outq[p * V + w] = key[u][w];
                        }
                        n_out += __popc(insm);
                    }
                }
            } else {
                for (uint32_t r0 = 0; r0 < m; r0 += 32) {
                    const uint32_t e = r0 + lane;
                    const bool act = e < m;
                    uint32_t key[V];
#pragma unroll
                    for (int w = 0; w < V; w++) key[w] = act ? q[e * V + w] : 0u;
                    int64_t hd;
                    const int code = act ? probe_status(T, key, fold<V>(T.salt, key), &hd) : -1;
                    const bool ins = act && code == INSERTED;
                    any_full |= act && code == TABLE_FULL;
                    const uint32_t insm = __ballot_sync(FULLMASK, ins);
                    if (ins) {
                        const uint32_t p = n_out + __popc(insm & lanemask_lt());
#pragma unroll
                        for (int w = 0; w < V; w++) outq[p * V + w] = key[w];
                    }
                    n_out += __popc(insm);
                }
            }
            if (__any_sync(FULLMASK, any_full) && lane == 0) atomicExch(&A.ctr[LV_FULL], 1ull);
            __syncwarp();
            if (n_out) flush_out<V>(A, outq, n_out);
            __syncwarp();
        }
    }
    trans = warp_sum(trans);
    expanded = warp_sum(expanded);
    probes = warp_sum(probes);
    if (lane == 0) {
        if (trans) atomicAdd(&A.ctr[LV_TRANS], trans);
        if (expanded) atomicAdd(&A.ctr[LV_EXP], expanded);
        if (probes) atomicAdd(&A.ctr[LV_PROBES], probes);
    }
}

template <int BW, int V>
__global__ void __launch_bounds__(256, GX_STAGED_MINB) k_level_staged(TableDesc T, NetDesc N, LevelArgs A) {
    level_staged_body<BW, V, false>(T, N, A, RouteArgs{});
}

struct LevelKernel {
    void (*fn)(TableDesc, NetDesc, LevelArgs);
    size_t fixed_smem;  // dynamic shared memory besides the dedup cache
};

template <int BW>
static LevelKernel pick_staged_v(int v) {
    switch (v) {
        case 1: return {k_level_staged<BW, 1>, StagedSmem<BW, 1>::FIXED};
        case 2: return {k_level_staged<BW, 2>, StagedSmem<BW, 2>::FIXED};
        case 4: return {k_level_staged<BW, 4>, StagedSmem<BW, 4>::FIXED};
    }
    return {nullptr, 0};
}

static LevelKernel pick_staged(const TableDesc& T) {
    switch (T.bw) {
        case 4: return pick_staged_v<4>((int)T.vlen);
        case 8: return pick_staged_v<8>((int)T.vlen);
        case 16: return pick_staged_v<16>((int)T.vlen);
        case 32: return pick_staged_v<32>((int)T.vlen);
    }
    return {nullptr, 0};
}

typedef void (*level_kernel_t)(TableDesc, NetDesc, LevelArgs);

template <int BW, int V>
static level_kernel_t pick_level_g(int g) {
    switch (g) {
        case 1: return k_level<BW, V, 1, true>;
        case 2: if (BW >= 8) return k_level<BW, V, (BW >= 8 ? 2 : 1), true>; break;
        case 4: if (BW >= 16) return k_level<BW, V, (BW >= 16 ? 4 : 1), true>; break;
        case 8: if (BW >= 32) return k_level<BW, V, (BW >= 32 ? 8 : 1), true>; break;
    }
    return nullptr;
}

template <int BW>
static level_kernel_t pick_level_v(int v, int g) {
    switch (v) {
        case 1: return pick_level_g<BW, 1>(g);
        case 2: return pick_level_g<BW, 2>(g);
        case 4: return pick_level_g<BW, 4>(g);
    }
    return nullptr;
}

static level_kernel_t pick_level_status(int v) {
    switch (v) {
#define GX_CASE(X) \
    case X: return k_level<0, X, 1, false>;
        GX_CASE(1) GX_CASE(2) GX_CASE(3) GX_CASE(4) GX_CASE(5) GX_CASE(6) GX_CASE(7) GX_CASE(8)
        GX_CASE(9) GX_CASE(10) GX_CASE(11) GX_CASE(12) GX_CASE(13) GX_CASE(14) GX_CASE(15)
        GX_CASE(16)
#undef GX_CASE
    }
    return nullptr;
}

int default_group(int bw);

static level_kernel_t pick_level(const TableDesc& T, int group) {
    if (T.mode == MODE_STATUS) return pick_level_status((int)T.vlen);
    const int g = group > 0 ? group : default_group((int)T.bw);
    switch (T.bw) {
        case 4: return pick_level_v<4>((int)T.vlen, g);
        case 8: return pick_level_v<8>((int)T.vlen, g);
        case 16: return pick_level_v<16>((int)T.vlen, g);
        case 32: return pick_level_v<32>((int)T.vlen, g);
    }
    return nullptr;
}

// ------------------------------------------------------------ gx_expand

template <int V>
__global__ void k_expand_count(NetDesc N, const uint32_t* __restrict__ states, uint64_t n,
                               unsigned long long* counts, uint32_t* nsucc) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t s[V];
#pragma unroll
    for (int w = 0; w < V; w++) s[w] = states[i * V + w];
    uint64_t c;
    nsucc[i] = expand_state<V, false>(N, s, &c, 0, 0, nullptr);
    counts[i] = c;
}

template <int V>
__global__ void k_expand_emit(NetDesc N, const uint32_t* __restrict__ states, uint64_t n,
                              const unsigned long long* offs, uint32_t* out, uint64_t cap) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t s[V];
#pragma unroll
    for (int w = 0; w < V; w++) s[w] = states[i * V + w];
    const unsigned long long o = offs[i];
    if (o >= cap) return;
    uint64_t c;
    expand_state<V, true>(N, s, &c, 0, (uint32_t)min((unsigned long long)UINT32_MAX, cap - o),
                          out + o * V);
}

typedef void (*count_kernel_t)(NetDesc, const uint32_t*, uint64_t, unsigned long long*, uint32_t*);
typedef void (*emit_kernel_t)(NetDesc, const uint32_t*, uint64_t, const unsigned long long*,
                              uint32_t*, uint64_t);

static count_kernel_t pick_count(int v) {
    switch (v) {
#define GX_CASE(X) \
    case X: return k_expand_count<X>;
        GX_CASE(1) GX_CASE(2) GX_CASE(3) GX_CASE(4) GX_CASE(5) GX_CASE(6) GX_CASE(7) GX_CASE(8)
        GX_CASE(9) GX_CASE(10) GX_CASE(11) GX_CASE(12) GX_CASE(13) GX_CASE(14) GX_CASE(15)
        GX_CASE(16)
#undef GX_CASE
    }
    return nullptr;
}

static emit_kernel_t pick_emit(int v) {
    switch (v) {
#define GX_CASE(X) \
    case X: return k_expand_emit<X>;
        GX_CASE(1) GX_CASE(2) GX_CASE(3) GX_CASE(4) GX_CASE(5) GX_CASE(6) GX_CASE(7) GX_CASE(8)
        GX_CASE(9) GX_CASE(10) GX_CASE(11) GX_CASE(12) GX_CASE(13) GX_CASE(14) GX_CASE(15)
        GX_CASE(16)
#undef GX_CASE
    }
    return nullptr;
}

// ------------------------------------------------- multi-GPU primitives

// owner-binning helpers over a flat successor buffer
__global__ void k_owner_hist(uint64_t salt, const uint32_t* __restrict__ keys, uint64_t n, int v,
                             int ranks, unsigned long long* counts) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int o = owner_of_mix(key_mix_rt(keys + i * v, v), ranks);
    atomicAdd(&counts[o], 1ull);
}

__global__ void k_owner_scatter(uint64_t salt, const uint32_t* __restrict__ keys, uint64_t n, int v,
                                int ranks, unsigned long long* cursor, uint32_t* out) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t* k = keys + i * v;
    const int o = owner_of_mix(key_mix_rt(k, v), ranks);
    const unsigned long long p = atomicAdd(&cursor[o], 1ull);
    for (int w = 0; w < v; w++) out[p * v + w] = k[w];
}

__global__ void k_owner_of(uint64_t salt, const uint32_t* __restrict__ keys, uint64_t n, int v,
                           int ranks, int32_t* out) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = owner_of_mix(key_mix_rt(keys + i * v, v), ranks);
}

// expand a frontier into a flat successor buffer (warp-aggregated append)
template <int V>
__global__ void __launch_bounds__(256) k_expand_flat(NetDesc N, const uint32_t* __restrict__ front,
                                                     uint64_t nfront, uint32_t* out, uint64_t cap,
                                                     unsigned long long* ctr, uint32_t* dl,
                                                     uint64_t dl_cap, int detect) {
    // ctr: [0] successors, [1] transitions, [2] deadlocks, [3] overflow
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    unsigned long long trans = 0;
    for (uint64_t base = warp * 32; base < nfront; base += nwarps * 32) {
        const uint64_t idx = base + lane;
        const bool has = idx < nfront;
        uint32_t s[V];
        if (has)
            load_state<V>(front + idx * V, s);
        else
#pragma unroll
            for (int w = 0; w < V; w++) s[w] = 0;
        uint64_t cnt = 0;
        uint32_t n = 0;
        if (has) {
            n = expand_state<V, false>(N, s, &cnt, 0, 0, nullptr);
            trans += cnt;
            if (cnt == 0 && detect) {
                unsigned long long p = atomicAdd(&ctr[2], 1ull);
                if (p < dl_cap) store_state<V>(dl + p * V, s);
            }
        }
        uint32_t incl = n;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(FULLMASK, incl, o);
            if (lane >= o) incl += y;
        }
        const uint32_t total = __shfl_sync(FULLMASK, incl, 31);
        unsigned long long b0 = 0;
        if (lane == 0 && total) b0 = atomicAdd(&ctr[0], (unsigned long long)total);
        b0 = __shfl_sync(FULLMASK, b0, 0);
        const unsigned long long my = b0 + incl - n;
        if (has && n) {
            if (my + n <= cap) {
                uint64_t dummy;
                expand_state<V, true>(N, s, &dummy, 0, n, out + my * V);
            } else {
                atomicExch(&ctr[3], 1ull);
            }
        }
    }
    trans = warp_sum(trans);
    if (lane == 0 && trans) atomicAdd(&ctr[1], trans);
}

typedef void (*flat_kernel_t)(NetDesc, const uint32_t*, uint64_t, uint32_t*, uint64_t,
                              unsigned long long*, uint32_t*, uint64_t, int);

static flat_kernel_t pick_flat(int v) {
    switch (v) {
#define GX_CASE(X) \
    case X: return k_expand_flat<X>;
        GX_CASE(1) GX_CASE(2) GX_CASE(3) GX_CASE(4) GX_CASE(5) GX_CASE(6) GX_CASE(7) GX_CASE(8)
        GX_CASE(9) GX_CASE(10) GX_CASE(11) GX_CASE(12) GX_CASE(13) GX_CASE(14) GX_CASE(15)
        GX_CASE(16)
#undef GX_CASE
    }
    return nullptr;
}

// FINDORPUT + append of INSERTED keys (the receive side of the exchange)
template <int V>
__device__ __forceinline__ void append_keys(unsigned long long* ctr, uint32_t* out, uint64_t cap,
                                            bool ins, const uint32_t* key) {
    const int lane = threadIdx.x & 31;
    const uint32_t insm = __ballot_sync(FULLMASK, ins);
    if (!insm) return;
    unsigned long long pos0 = 0;
    if (lane == 0) pos0 = atomicAdd(&ctr[0], (unsigned long long)__popc(insm));
    pos0 = __shfl_sync(FULLMASK, pos0, 0);
    if (ins) {
        const unsigned long long p = pos0 + __popc(insm & lanemask_lt());
        if (p < cap)
            store_state<V>(out + p * V, key);
        else
            atomicExch(&ctr[2], 1ull);
    }
}

// FINDORPUT + append of INSERTED keys (the receive side of the exchange)
template <int BW, int V, int G, bool MARK>
__global__ void __launch_bounds__(256) k_insert_append(TableDesc T, const uint32_t* __restrict__ keys,
                                                       uint64_t n, uint32_t* out, uint64_t cap,
                                                       unsigned long long* ctr) {
    // ctr: [0] appended, [1] table full, [2] overflow
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    bool any_full = false;
    if constexpr (MARK) {
        using S = ProbeShape<BW, G>;
        const bool leader = (lane & (G - 1)) == 0;
        for (uint64_t base = warp * S::KB; base < n; base += nwarps * S::KB) {
            uint32_t own_key[S::M][V];
            bool own_act[S::M];
#pragma unroll
            for (int mm = 0; mm < S::M; mm++) {
                const uint64_t e = base + lane + 32 * mm;
                own_act[mm] = e < n;
#pragma unroll
                for (int w = 0; w < V; w++) own_key[mm][w] = own_act[mm] ? keys[e * V + w] : 0u;
            }
            uint32_t key[S::U][V];
            bool act[S::U];
            int code[S::U];
            int64_t hd[S::U];
            probe_batch<BW, V, G>(T, own_key, own_act, key, act, code, hd);
#pragma unroll
            for (int u = 0; u < S::U; u++) {
                any_full |= leader && act[u] && code[u] == TABLE_FULL;
                append_keys<V>(ctr, out, cap, leader && act[u] && code[u] == INSERTED, key[u]);
            }
        }
    } else {
        for (uint64_t base = warp * 32; base < n; base += nwarps * 32) {
            const uint64_t e = base + lane;
            const bool act = e < n;
            uint32_t key[V];
#pragma unroll
            for (int w = 0; w < V; w++) key[w] = act ? keys[e * V + w] : 0u;
            int64_t hd;
            const int code = act ? probe_status(T, key, fold<V>(T.salt, key), &hd) : -1;
            any_full |= act && code == TABLE_FULL;
            append_keys<V>(ctr, out, cap, act && code == INSERTED, key);
        }
    }
    if (__any_sync(FULLMASK, any_full) && lane == 0) atomicExch(&ctr[1], 1ull);
}

typedef void (*append_kernel_t)(TableDesc, const uint32_t*, uint64_t, uint32_t*, uint64_t,
                                unsigned long long*);

template <int BW, int V>
static append_kernel_t pick_append_g(int g) {
    switch (g) {
        case 1: return k_insert_append<BW, V, 1, true>;
        case 2: if (BW >= 8) return k_insert_append<BW, V, (BW >= 8 ? 2 : 1), true>; break;
        case 4: if (BW >= 16) return k_insert_append<BW, V, (BW >= 16 ? 4 : 1), true>; break;
        case 8: if (BW >= 32) return k_insert_append<BW, V, (BW >= 32 ? 8 : 1), true>; break;
    }
    return nullptr;
}

template <int BW>
static append_kernel_t pick_append_v(int v, int g) {
    switch (v) {
        case 1: return pick_append_g<BW, 1>(g);
        case 2: return pick_append_g<BW, 2>(g);
        case 4: return pick_append_g<BW, 4>(g);
    }
    return nullptr;
}

static append_kernel_t pick_append(const TableDesc& T, int group) {
    if (T.mode == MODE_STATUS) {
        switch (T.vlen) {
#define GX_CASE(X) \
    case X: return k_insert_append<0, X, 1, false>;
            GX_CASE(1) GX_CASE(2) GX_CASE(3) GX_CASE(4) GX_CASE(5) GX_CASE(6) GX_CASE(7) GX_CASE(8)
            GX_CASE(9) GX_CASE(10) GX_CASE(11) GX_CASE(12) GX_CASE(13) GX_CASE(14) GX_CASE(15)
            GX_CASE(16)
#undef GX_CASE
        }
        return nullptr;
    }
    const int g = group > 0 ? group : default_group((int)T.bw);
    switch (T.bw) {
        case 4: return pick_append_v<4>((int)T.vlen, g);
        case 8: return pick_append_v<8>((int)T.vlen, g);
        case 16: return pick_append_v<16>((int)T.vlen, g);
        case 32: return pick_append_v<32>((int)T.vlen, g);
    }
    return nullptr;
}

// ------------------------------------------------------------ benchmark

template <int BW, int V, int G, bool MARK>
__global__ void __launch_bounds__(256) k_bench(TableDesc T, BenchArgs B) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    unsigned long long ins = 0, full = 0;
    if constexpr (MARK) {
        using S = ProbeShape<BW, G>;
        const bool leader = (lane & (G - 1)) == 0;
        for (uint64_t base = warp * S::KB; base < B.total; base += nwarps * S::KB) {
            uint32_t own_key[S::M][V];
            bool own_act[S::M];
#pragma unroll
            for (int mm = 0; mm < S::M; mm++) {
                const uint64_t e = base + lane + 32 * mm;
                own_act[mm] = e < B.total;
                if (own_act[mm])
                    bench_key<V>(B, e, own_key[mm]);
                else
#pragma unroll
                    for (int w = 0; w < V; w++) own_key[mm][w] = 0;
            }
            uint32_t key[S::U][V];
            bool act[S::U];
            int code[S::U];
            int64_t hd[S::U];
            probe_batch<BW, V, G>(T, own_key, own_act, key, act, code, hd);
#pragma unroll
            for (int u = 0; u < S::U; u++) {
                ins += leader && act[u] && code[u] == INSERTED;
                full += leader && act[u] && code[u] == TABLE_FULL;
            }
        }
    } else {
        for (uint64_t e = warp * 32 + lane; e < B.total + 31; e += nwarps * 32) {
            if (e >= B.total) break;
            uint32_t key[V];
            bench_key<V>(B, e, key);
            int64_t hd;
            const int code = probe_status(T, key, fold<V>(T.salt, key), &hd);
            ins += code == INSERTED;
            full += code == TABLE_FULL;
        }
    }
    ins = warp_sum(ins);
    full = warp_sum(full);
    if (lane == 0) {
        if (ins) atomicAdd(&B.ctr[0], ins);
        if (full) atomicAdd(&B.ctr[1], full);
    }
}

typedef void (*bench_kernel_t)(TableDesc, BenchArgs);

#ifndef GX_BENCH_BATCH
#define GX_BENCH_BATCH 512  // keys generated per warp per probe call
#endif

// The same benchmark on the staged probe (the level kernel's FINDORPUT):
// each warp generates KB keys into its shared-memory queue and resolves
// them with probe_staged.  Counts INSERTED / TABLE_FULL.
template <int BW, int V>
__global__ void __launch_bounds__(256, 2) k_bench_staged(TableDesc T, BenchArgs B) {
    using S = Staged<BW, V>;
    constexpr int KB = S::KB;
    constexpr int BQ = GX_BENCH_BATCH;  // keys per warp per probe call (the refill probe keeps 32 lanes busy)
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    uint32_t* q = reinterpret_cast<uint32_t*>(smem) + wid * (BQ * V);
    unsigned long long* sbkt = reinterpret_cast<unsigned long long*>(smem + 8ull * BQ * V * 4) + wid * S::SB_STRIDE;
    uint4* stage = reinterpret_cast<uint4*>(smem + 8ull * BQ * V * 4 + 8ull * S::SB_STRIDE * 8 +
                                            (size_t)wid * S::STAGE_BYTES);
    staged_init(sbkt, KB);
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    unsigned long long ins = 0, full = 0, loads = 0;
    for (uint64_t base = warp * BQ; base < B.total; base += nwarps * BQ) {
        const uint32_t m = (uint32_t)min((uint64_t)BQ, B.total - base);
        for (uint32_t k = lane; k < m; k += 32) {
            uint32_t key[V];
            bench_key<V>(B, base + k, key);
#pragma unroll
            for (int w = 0; w < V; w++) q[k * V + w] = key[w];
        }
        __syncwarp();
        uint32_t f = 0, np = 0;
        const uint32_t n_ins = probe_staged<BW, V>(T, q, m, stage, sbkt, &f, &np);
        ins += lane == 0 ? n_ins : 0;
        full += f;  // keys that hit TABLE_FULL
        loads += np;
        __syncwarp();
    }
    ins = warp_sum(ins);
    full = warp_sum(full);
    loads = warp_sum(loads);
    if (lane == 0) {
        if (ins) atomicAdd(&B.ctr[0], ins);
        if (full) atomicAdd(&B.ctr[1], full);
        if (loads) atomicAdd(&B.ctr[2], loads);
    }
}

template <int BW, int V>
static size_t bench_staged_smem() {
    using S = Staged<BW, V>;
    return 8ull * GX_BENCH_BATCH * V * 4 + 8ull * S::SB_STRIDE * 8 + 8ull * S::STAGE_BYTES;
}

struct BenchKernel {
    void (*fn)(TableDesc, BenchArgs);
    size_t smem;
};

template <int BW>
static BenchKernel pick_bench_staged_v(int v) {
    switch (v) {
        case 1: return {k_bench_staged<BW, 1>, bench_staged_smem<BW, 1>()};
        case 2: return {k_bench_staged<BW, 2>, bench_staged_smem<BW, 2>()};
        case 4: return {k_bench_staged<BW, 4>, bench_staged_smem<BW, 4>()};
    }
    return {nullptr, 0};
}

static BenchKernel pick_bench_staged(const TableDesc& T) {
    switch (T.bw) {
        case 4: return pick_bench_staged_v<4>((int)T.vlen);
        case 8: return pick_bench_staged_v<8>((int)T.vlen);
        case 16: return pick_bench_staged_v<16>((int)T.vlen);
        case 32: return pick_bench_staged_v<32>((int)T.vlen);
    }
    return {nullptr, 0};
}

template <int BW, int V>
static bench_kernel_t pick_bench_g(int g) {
    switch (g) {
        case 1: return k_bench<BW, V, 1, true>;
        case 2: if (BW >= 8) return k_bench<BW, V, (BW >= 8 ? 2 : 1), true>; break;
        case 4: if (BW >= 16) return k_bench<BW, V, (BW >= 16 ? 4 : 1), true>; break;
        case 8: if (BW >= 32) return k_bench<BW, V, (BW >= 32 ? 8 : 1), true>; break;
    }
    return nullptr;
}

template <int BW>
static bench_kernel_t pick_bench_v(int v, int g) {
    switch (v) {
        case 1: return pick_bench_g<BW, 1>(g);
        case 2: return pick_bench_g<BW, 2>(g);
        case 4: return pick_bench_g<BW, 4>(g);
    }
    return nullptr;
}

static bench_kernel_t pick_bench(const TableDesc& T, int group) {
    if (T.mode == MODE_STATUS) {
        switch (T.vlen) {
            case 1: return k_bench<0, 1, 1, false>;
            case 2: return k_bench<0, 2, 1, false>;
            case 3: return k_bench<0, 3, 1, false>;
            case 4: return k_bench<0, 4, 1, false>;
        }
        return nullptr;
    }
    const int g = group > 0 ? group : default_group((int)T.bw);
    switch (T.bw) {
        case 4: return pick_bench_v<4>((int)T.vlen, g);
        case 8: return pick_bench_v<8>((int)T.vlen, g);
        case 16: return pick_bench_v<16>((int)T.vlen, g);
        case 32: return pick_bench_v<32>((int)T.vlen, g);
    }
    return nullptr;
}

// composite-order comparison of two packed vectors (unpack, then
// lexicographic over processes: sorted() of state tuples, explore.py:361-367)
bool composite_less(const gx_net* n, const uint32_t* a, const uint32_t* b) {
    for (uint32_t i = 0; i < n->nproc; i++) {
        const uint4 p = n->proc_host[i];
        const uint32_t x = (a[p.x] >> p.y) & p.z, y = (b[p.x] >> p.y) & p.z;
        if (x != y) return x < y;
    }
    return false;
}

void keep_smallest(const gx_net* n, std::vector<uint32_t>& kept, const uint32_t* add,
                          uint64_t cnt) {
    const uint32_t v = n->vlen;
    const uint64_t have = kept.size() / v;
    std::vector<uint64_t> idx(have + cnt);
    std::vector<uint32_t> all(kept);
    all.insert(all.end(), add, add + cnt * v);
    for (uint64_t i = 0; i < idx.size(); i++) idx[i] = i;
    std::sort(idx.begin(), idx.end(), [&](uint64_t x, uint64_t y) {
        return composite_less(n, all.data() + x * v, all.data() + y * v);
    });
    const uint64_t keep = std::min<uint64_t>(idx.size(), GX_DEADLOCK_KEEP);
    kept.resize(keep * v);
    for (uint64_t i = 0; i < keep; i++)
        memcpy(kept.data() + i * v, all.data() + idx[i] * v, sizeof(uint32_t) * v);
}

static int persistent_grid() { return sm_count() * 8; }

// Deadlock states of frontier F[0, n) (count == 0), recorded in dl with the
// counter cell (the fallback of a level that found more deadlocks than its
// record buffer holds; explore.py:220-226 keeps the 100 smallest of ALL).
template <int V>
__global__ void k_dl_scan(NetDesc N, const uint32_t* __restrict__ F, uint64_t n, uint32_t* dl,
                          unsigned long long* cell) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t s[V];
    load_state<V>(F + i * V, s);
    uint64_t c;
    expand_state<V, false>(N, s, &c, 0, 0, nullptr);
    if (c == 0) store_state<V>(dl + atomicAdd(cell, 1ull) * V, s);
}

typedef void (*dl_scan_t)(NetDesc, const uint32_t*, uint64_t, uint32_t*, unsigned long long*);

static dl_scan_t pick_dl_scan(int v) {
    switch (v) {
#define GX_CASE(X) \
    case X: return k_dl_scan<X>;
        GX_CASE(1) GX_CASE(2) GX_CASE(3) GX_CASE(4) GX_CASE(5) GX_CASE(6) GX_CASE(7) GX_CASE(8)
        GX_CASE(9) GX_CASE(10) GX_CASE(11) GX_CASE(12) GX_CASE(13) GX_CASE(14) GX_CASE(15)
        GX_CASE(16)
#undef GX_CASE
    }
    return nullptr;
}

// Re-expand the frontier F[0, nF) in chunks of dl_cap states (so no chunk
// can overflow the record buffer dl) and merge every chunk's deadlocks into
// `kept`: exact 100 smallest however many deadlocks one level has.
int rescan_deadlocks(const gx_net* n, const uint32_t* F, uint64_t nF, uint32_t* dl, uint64_t dl_cap,
                     unsigned long long* cell, cudaStream_t st, std::vector<uint32_t>& kept) {
    const uint32_t v = n->vlen;
    dl_scan_t k = pick_dl_scan((int)v);
    std::vector<uint32_t> host;
    for (uint64_t b = 0; b < nF; b += dl_cap) {
        const uint64_t m = std::min<uint64_t>(dl_cap, nF - b);
        GX_CUDA(cudaMemsetAsync(cell, 0, 8, st));
        k<<<(int)((m + 255) / 256), 256, 0, st>>>(n->d, F + b * v, m, dl, cell);
        GX_LAUNCHED();
        unsigned long long c = 0;
        GX_CUDA(cudaMemcpyAsync(&c, cell, 8, cudaMemcpyDeviceToHost, st));
        GX_CUDA(cudaStreamSynchronize(st));
        if (!c) continue;
        host.resize(c * v);
        GX_CUDA(cudaMemcpyAsync(host.data(), dl, sizeof(uint32_t) * c * v, cudaMemcpyDeviceToHost, st));
        GX_CUDA(cudaStreamSynchronize(st));
        keep_smallest(n, kept, host.data(), c);
    }
    return GX_OK;
}

}  // namespace gx

using namespace gx;

// ===================================================================== C ABI

extern "C" {

int gx_net_create(const gx_network_csr* c, void* stream, gx_net** out) {
    *out = nullptr;
    if (c->vlen < 1 || c->vlen > GX_MAXV) {
        set_error("vector length %u outside 1..%d", c->vlen, GX_MAXV);
        return GX_EINPUT;
    }
    if (c->n_proc != 4ull * c->nproc || c->n_rules != 4ull * c->nrules || c->n_qtab % 4 ||
        c->n_parts % 4 || c->n_rq % 2 || c->n_trig < 1 || c->n_dedup < 1) {
        set_error("malformed network CSR (section sizes)");
        return GX_EINPUT;
    }
    gx_net* n = new gx_net();
    n->stream = (cudaStream_t)stream;
    n->vlen = c->vlen;
    n->nproc = c->nproc;
    n->initial.assign(c->initial, c->initial + c->vlen);
    n->proc_host.resize(c->nproc);
    memcpy(n->proc_host.data(), c->proc, sizeof(uint32_t) * c->n_proc);
    // one blob, each section 16-byte aligned
    const uint32_t* src[9] = {c->proc, c->qtab, c->im_dst, c->trig, c->rules,
                              c->parts, c->rq, c->rdst, c->dedup};
    const uint64_t len[9] = {c->n_proc, c->n_qtab, c->n_im_dst, c->n_trig, c->n_rules,
                             c->n_parts, c->n_rq, c->n_rdst, c->n_dedup};
    uint64_t off[10];
    off[0] = 0;
    for (int i = 0; i < 9; i++) off[i + 1] = off[i] + ((len[i] + 3) & ~3ull) + 4;
    std::vector<uint32_t> blob(off[9] + 4, 0u);
    for (int i = 0; i < 9; i++)
        if (len[i]) memcpy(blob.data() + off[i], src[i], sizeof(uint32_t) * len[i]);
    // pack each qtab entry's trigger count next to its offset when all
    // offsets fit in 24 bits (255 = read the count from the list)
    bool packed = c->n_trig < (1ull << 24);
    if (packed) {
        uint32_t* q = blob.data() + off[1];
        for (uint64_t e = 0; e + 3 < c->n_qtab; e += 4) {
            const uint32_t toff = q[e + 3];
            const uint32_t nt = c->trig[toff];
            q[e + 3] = toff | (std::min<uint32_t>(nt, 255u) << 24);
        }
    }
    // per rule, the bits its participants occupy in each of the first 4
    // words (vlen <= 4): rule_generates rejects most dedup candidates with
    // one 16-byte load instead of walking the participant list
    const uint64_t rm_off = blob.size() + ((4 - blob.size() % 4) % 4);
    blob.resize(rm_off + 4ull * std::max<uint32_t>(c->nrules, 1), 0u);
    if (c->vlen <= 4) {
        for (uint32_t r = 0; r < c->nrules; r++) {
            const uint32_t np_ = c->rules[4 * r], po = c->rules[4 * r + 1];
            for (uint32_t k = 0; k < np_; k++) {
                const uint32_t* pt = c->parts + 4ull * (po + k);
                if (pt[1] < 4) blob[rm_off + 4ull * r + pt[1]] |= pt[3] << pt[2];
            }
        }
    }
    // process groups for the grouped expansion (gx_internal.h NetDesc):
    // consecutive processes with adjacent fields in one word, at most
    // GX_GROUP_BITS bits together; one table entry per joint field code
    const uint32_t P = c->nproc;
    std::vector<uint32_t> nst(P);
    for (uint32_t k = 0; k < P; k++) {
        const uint32_t qb = c->proc[4 * k + 3];
        const uint32_t qe = k + 1 < P ? c->proc[4 * (k + 1) + 3] : (uint32_t)(c->n_qtab / 4);
        nst[k] = qe - qb;
    }
    struct Grp { uint32_t word, shift, bits, p0, np; };
    std::vector<Grp> grps;
    for (uint32_t k = 0; k < P; k++) {
        const uint32_t w = c->proc[4 * k], sh = c->proc[4 * k + 1], bits = __builtin_popcount(c->proc[4 * k + 2]);
        if (!grps.empty()) {
            Grp& g = grps.back();
            if (g.word == w && g.shift + g.bits == sh && g.bits + bits <= GX_GROUP_BITS && g.np < 24) {
                g.bits += bits;
                g.np++;
                continue;
            }
        }
        grps.push_back(Grp{w, sh, bits, k, 1});
    }
    std::vector<uint32_t> gtab, gdelta;
    const bool grouped = GX_GROUP_BITS > 0 && grps.size() < P && grps.size() <= GX_GROUP_INLINE;
    if (grouped) {
        for (const Grp& g : grps) {
            for (uint32_t code = 0; code < (1u << g.bits); code++) {
                uint32_t cnt = 0, ns = 0, tm = 0;
                const uint32_t off = (uint32_t)gdelta.size();
                bool valid = true;
                for (uint32_t k = 0; k < g.np && valid; k++) {
                    const uint32_t p = g.p0 + k;
                    const uint32_t sh = c->proc[4 * p + 1], mask = c->proc[4 * p + 2], qb = c->proc[4 * p + 3];
                    const uint32_t v = (code >> (sh - g.shift)) & mask;
                    if (v >= nst[p]) {
                        valid = false;
                        break;
                    }
                    const uint32_t* q = c->qtab + 4ull * (qb + v);  // {im_off, im_n, im_cnt, trig_off}
                    cnt += q[2];
                    for (uint32_t d = 0; d < q[1]; d++) gdelta.push_back((v ^ c->im_dst[q[0] + d]) << sh);
                    ns += q[1];
                    if (c->trig[q[3]] != 0) tm |= 1u << k;
                }
                if (!valid) {
                    gdelta.resize(off);
                    cnt = ns = tm = 0;
                }
                gtab.insert(gtab.end(), {cnt, ns, off, tm});
            }
        }
    }
    const uint64_t gt_off = blob.size();
    blob.insert(blob.end(), gtab.begin(), gtab.end());
    const uint64_t gd_off = blob.size();
    blob.insert(blob.end(), gdelta.begin(), gdelta.end());
    blob.push_back(0u);
    cudaError_t e = cudaMalloc(&n->d_blob, sizeof(uint32_t) * blob.size());
    if (e == cudaSuccess) e = cudaMalloc(&n->d_initial, sizeof(uint32_t) * 16);
    if (e != cudaSuccess) {
        set_error("network upload failed: %s", cudaGetErrorString(e));
        delete n;
        return GX_EINTERNAL;
    }
    GX_CUDA(cudaMemcpyAsync(n->d_blob, blob.data(), sizeof(uint32_t) * blob.size(),
                            cudaMemcpyHostToDevice, n->stream));
    GX_CUDA(cudaMemcpyAsync(n->d_initial, c->initial, sizeof(uint32_t) * c->vlen,
                            cudaMemcpyHostToDevice, n->stream));
    GX_CUDA(cudaStreamSynchronize(n->stream));
    NetDesc& d = n->d;
    d.proc = (const uint4*)(n->d_blob + off[0]);
    d.qtab = (const uint4*)(n->d_blob + off[1]);
    d.im_dst = n->d_blob + off[2];
    d.trig = n->d_blob + off[3];
    d.rules = (const uint4*)(n->d_blob + off[4]);
    d.parts = (const uint4*)(n->d_blob + off[5]);
    d.rq = (const uint2*)(n->d_blob + off[6]);
    d.rdst = n->d_blob + off[7];
    d.dedup = n->d_blob + off[8];
    d.rmask = c->vlen <= 4 ? (const uint4*)(n->d_blob + rm_off) : nullptr;
    d.nproc = c->nproc;
    d.nrules = c->nrules;
    d.vlen = c->vlen;
    d.trig_packed = packed ? 1u : 0u;
    memset(d.proc_c, 0, sizeof d.proc_c);
    for (uint32_t i = 0; i < c->nproc && i < GX_PROC_INLINE; i++)
        d.proc_c[i] = make_uint4(c->proc[4 * i], c->proc[4 * i + 1], c->proc[4 * i + 2], c->proc[4 * i + 3]);
    d.gtab = (const uint4*)(n->d_blob + gt_off);
    d.gdelta = n->d_blob + gd_off;
    d.ngroups = grouped ? (uint32_t)grps.size() : 0u;
    memset(d.gdesc, 0, sizeof d.gdesc);
    uint32_t base = 0;
    for (size_t g = 0; grouped && g < grps.size(); g++) {
        d.gdesc[g] = make_uint4(grps[g].word | grps[g].p0 << 8 | grps[g].np << 24, grps[g].shift,
                                (1u << grps[g].bits) - 1u, base);
        base += 1u << grps[g].bits;
    }
    *out = n;
    return GX_OK;
}

int gx_net_destroy(gx_net* n) {
    if (!n) return GX_OK;
    cudaStreamSynchronize(n->stream);
    cudaFree(n->d_blob);
    cudaFree(n->d_initial);
    n->scratch.release();
    n->dl.release();
    delete n;
    return GX_OK;
}

int gx_expand(gx_net* n, const uint32_t* states, uint64_t ns, uint64_t* counts, uint32_t* nsucc,
              uint32_t* succ, uint64_t cap, uint64_t* total) {
    const uint64_t v = n->vlen;
    if (ns == 0) {
        if (total) *total = 0;
        return GX_OK;
    }
    // scratch: states | counts | nsucc | offsets | out
    const uint64_t b_states = sizeof(uint32_t) * ns * v, b_counts = 8 * ns, b_n = 4 * ns,
                   b_offs = 8 * ns;
    const uint64_t b_out = sizeof(uint32_t) * std::max<uint64_t>(cap, 1) * v;
    int rc = n->scratch.ensure(b_states + b_counts + b_n + b_offs + b_out + 64);
    if (rc) return rc;
    char* base = (char*)n->scratch.p;
    uint32_t* d_states = (uint32_t*)base;
    unsigned long long* d_counts = (unsigned long long*)(base + ((b_states + 15) & ~15ull));
    uint32_t* d_n = (uint32_t*)((char*)d_counts + b_counts);
    unsigned long long* d_offs = (unsigned long long*)((char*)d_n + ((b_n + 15) & ~15ull));
    uint32_t* d_out = (uint32_t*)((char*)d_offs + b_offs);
    GX_CUDA(cudaMemcpyAsync(d_states, states, b_states, cudaMemcpyHostToDevice, n->stream));
    pick_count((int)v)<<<(int)((ns + 127) / 128), 128, 0, n->stream>>>(n->d, d_states, ns, d_counts, d_n);
    GX_LAUNCHED();
    std::vector<unsigned long long> hc(ns);
    std::vector<uint32_t> hn(ns);
    GX_CUDA(cudaMemcpyAsync(hc.data(), d_counts, b_counts, cudaMemcpyDeviceToHost, n->stream));
    GX_CUDA(cudaMemcpyAsync(hn.data(), d_n, b_n, cudaMemcpyDeviceToHost, n->stream));
    GX_CUDA(cudaStreamSynchronize(n->stream));
    std::vector<unsigned long long> offs(ns);
    unsigned long long tot = 0;
    for (uint64_t i = 0; i < ns; i++) {
        offs[i] = tot;
        tot += hn[i];
        if (counts) counts[i] = hc[i];
        if (nsucc) nsucc[i] = hn[i];
    }
    if (total) *total = tot;
    if (succ && cap) {
        GX_CUDA(cudaMemcpyAsync(d_offs, offs.data(), b_offs, cudaMemcpyHostToDevice, n->stream));
        pick_emit((int)v)<<<(int)((ns + 127) / 128), 128, 0, n->stream>>>(n->d, d_states, ns, d_offs,
                                                                          d_out, cap);
        GX_LAUNCHED();
        GX_CUDA(cudaMemcpyAsync(succ, d_out, sizeof(uint32_t) * std::min<uint64_t>(cap, tot) * v,
                                cudaMemcpyDeviceToHost, n->stream));
        GX_CUDA(cudaStreamSynchronize(n->stream));
    }
    return GX_OK;
}

int gx_explore(gx_net* n, gx_table* t, const gx_explore_cfg* cfg, gx_report* rep, uint32_t* deadlocks) {
    memset(rep, 0, sizeof *rep);
    const TableDesc& T = t->d;
    const uint32_t v = n->vlen;
    if (T.vlen != v) {
        set_error("table vector length %u != network vector length %u", T.vlen, v);
        return GX_EINPUT;
    }
    cudaStream_t st = t->stream;
    const uint64_t launches0 = gx_kernel_launches();
    // probe_group 0 (auto) on in-band tables: the shared-memory staged
    // level kernel; 1/2/4/8: the register-group kernel with that many lanes
    // per bucket; status-byte tables: one lane per key
    const bool staged = T.mode == MODE_MARK && cfg->probe_group == 0;
    LevelKernel LK = staged ? pick_staged(T) : LevelKernel{pick_level(T, cfg->probe_group), 0};
    level_kernel_t lk = LK.fn;
    if (!lk) {
        set_error("no level kernel for bw=%u vlen=%u group=%d", T.bw, v, cfg->probe_group);
        return GX_EINPUT;
    }
    // block-local dedup cache: cache_slots, at most GX_CACHE_MAX_SLOTS and
    // what keeps GX_STAGED_MINB blocks per SM resident (any count; only for
    // in-band tables with vlen <= 2)
    uint32_t cslots = 0;
    if (cfg->cache_slots > 0 && T.mode == MODE_MARK && v <= 2) {
        const size_t budget = STAGED_SMEM_BUDGET;
        const size_t fixed = LK.fixed_smem + (staged ? 0 : 2 * 8 * QWORDS_REG * 4);
        const size_t room = budget > fixed ? (budget - fixed) / 8 : 0;
        cslots = (uint32_t)std::min<size_t>({(size_t)cfg->cache_slots, (size_t)GX_CACHE_MAX_SLOTS, room});
        if (cslots < 32) cslots = 0;
    }
    const size_t csmem = LK.fixed_smem + sizeof(unsigned long long) * cslots;
    GX_CUDA(cudaFuncSetAttribute((const void*)lk, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)csmem));
    int rc = gx_table_clear(t);
    if (rc) return rc;
    // GPU-wide L2 dedup filter (in-band tables, vlen <= 2), cleared per search
    uint64_t gslots = 0;
    if (cfg->filter_log2 > 0 && T.mode == MODE_MARK && v <= 2) {
        gslots = 1ull << std::min(cfg->filter_log2, 28);
        rc = t->gfilter.ensure(8 * gslots);
        if (rc) return rc;
        GX_CUDA(cudaMemsetAsync(t->gfilter.p, 0, 8 * gslots, st));
    }
    // frontier buffer: two-ended, capacity C vectors
    uint64_t C = cfg->frontier_capacity;
    if (C == 0) {
        size_t fr = 0, tot = 0;
        GX_CUDA(cudaMemGetInfo(&fr, &tot));
        const uint64_t reserve = 512ull << 20;
        // the buffer we already hold counts as available (it is reused)
        const uint64_t have = (uint64_t)fr + t->aux2.bytes;
        const uint64_t avail = have > reserve + (64ull << 20) ? have - reserve : (64ull << 20);
        C = std::min<uint64_t>(t->total_slots + 2, avail * 9 / 10 / (4ull * v));
        if (C < 1024) C = 1024;
    }
    rc = t->aux2.ensure(sizeof(uint32_t) * C * v);
    if (rc) return rc;
    uint32_t* fb = (uint32_t*)t->aux2.p;
    const uint64_t dl_cap = 1 << 16;
    rc = n->dl.ensure(sizeof(uint32_t) * dl_cap * v);
    if (rc) return rc;
    cudaEvent_t e0, e1;
    GX_CUDA(cudaEventCreate(&e0));
    GX_CUDA(cudaEventCreate(&e1));
    GX_CUDA(cudaEventRecord(e0, st));
    // initial state (explore.py:311-315)
    rc = t->codes.ensure(16);
    if (rc) return rc;
    rc = table_find_or_put_dev(t, n->d_initial, 1, (uint8_t*)t->codes.p, nullptr, 0, cfg->probe_group);
    if (rc) return rc;
    GX_CUDA(cudaMemcpyAsync(fb, n->d_initial, sizeof(uint32_t) * v, cudaMemcpyDeviceToDevice, st));
    uint8_t code0 = 0;
    GX_CUDA(cudaMemcpyAsync(&code0, t->codes.p, 1, cudaMemcpyDeviceToHost, st));
    GX_CUDA(cudaStreamSynchronize(st));
    unsigned long long* ctr = (unsigned long long*)t->d_ctr;
    unsigned long long* hc = (unsigned long long*)t->h_ctr;
    std::vector<uint32_t> kept;
    std::vector<uint32_t> dlhost;
    uint64_t rounds = 0, states = 0, max_front = 0;
    int outcome = GX_COMPLETE;
    const uint32_t* pending = nullptr;  // last produced, unexpanded frontier
    uint64_t n_pending = 0;
    if (code0 == TABLE_FULL) {
        outcome = GX_OUTCOME_TABLE_FULL;
    } else {
        states = 1;
        // F at the left end, F' grows from the right end (and vice versa)
        const uint32_t* F = fb;
        uint64_t nF = 1;
        int rev = 1;
        unsigned long long new_base = 0, dl_base = 0;
        // exactly the resident blocks: one wave, so every block's strided
        // share of the frontier runs concurrently (no partial last wave)
        int resident = 0;
        GX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, lk, 256, csmem));
        const int grid = sm_count() * std::max(resident, 1);
        cudaEvent_t la, lb;
        GX_CUDA(cudaEventCreate(&la));
        GX_CUDA(cudaEventCreate(&lb));
        for (;;) {
            const uint64_t claims = nF;
            max_front = std::max<uint64_t>(max_front, nF);
            uint64_t nnew = 0;
            const uint32_t* Fn = nullptr;
            if (claims) {
                LevelArgs A;
                A.front = F;
                A.nfront = nF;
                A.out = fb;
                A.out_cap = C;
                A.out_limit = C - nF;
                A.out_rev = rev;
                A.detect = cfg->detect_deadlocks;
                A.ctr = ctr;
                A.new_base = new_base;
                A.dl_base = dl_base;
                A.dl = (uint32_t*)n->dl.p;
                A.dl_cap = dl_cap;
                A.cache_mask = cslots ? cslots - 1 : 0;
                A.gfilter_mask = gslots ? (uint32_t)(gslots - 1) : 0;
                A.gfilter = (unsigned long long*)t->gfilter.p;
                const uint64_t want = (nF + 31) / 32;  // warps
                const int g = (int)std::min<uint64_t>((uint64_t)grid, (want + 7) / 8);
                GX_CUDA(cudaEventRecord(la, st));
                lk<<<g, 256, csmem, st>>>(T, n->d, A);
                GX_LAUNCHED();
                GX_CUDA(cudaEventRecord(lb, st));
                rep->levels_launched++;
            }
            GX_CUDA(cudaMemcpyAsync(hc, ctr, sizeof(uint64_t) * CTR_N, cudaMemcpyDeviceToHost, st));
            GX_CUDA(cudaStreamSynchronize(st));
            if (claims) {
                float lms = 0;
                GX_CUDA(cudaEventElapsedTime(&lms, la, lb));
                rep->level_ms += lms;
            }
            nnew = hc[LV_NEW] - new_base;
            new_base = hc[LV_NEW];
            if (hc[LV_DL] > dl_base) {
                const uint64_t d = hc[LV_DL] - dl_base;
                if (d <= dl_cap) {
                    dlhost.resize(d * v);
                    GX_CUDA(cudaMemcpyAsync(dlhost.data(), n->dl.p, sizeof(uint32_t) * d * v,
                                            cudaMemcpyDeviceToHost, st));
                    GX_CUDA(cudaStreamSynchronize(st));
                    keep_smallest(n, kept, dlhost.data(), d);
                } else {  // the buffer overflowed: re-derive this level's deadlocks in chunks
                    rc = rescan_deadlocks(n, F, nF, (uint32_t*)n->dl.p, dl_cap, ctr + CTR_SCRATCH, st, kept);
                    if (rc) return rc;
                }
                dl_base = hc[LV_DL];
            }
            if (hc[LV_OVF]) {
                set_error("frontier capacity (%llu vectors) exceeded; raise frontier_capacity",
                          (unsigned long long)C);
                cudaEventDestroy(e0);
                cudaEventDestroy(e1);
                return GX_EINTERNAL;
            }
            states += nnew;
            Fn = rev ? fb + (C - nnew) * v : fb;
            rounds++;
            pending = Fn;
            n_pending = nnew;
            if (hc[LV_FULL]) {
                outcome = GX_OUTCOME_TABLE_FULL;
                break;
            }
            if (claims == 0) break;
            if (cfg->max_iterations >= 0 && rounds >= (uint64_t)cfg->max_iterations) {
                outcome = GX_ITERATION_CAP;
                break;
            }
            F = Fn;
            nF = nnew;
            rev ^= 1;
        }
        cudaEventDestroy(la);
        cudaEventDestroy(lb);
    }
    GX_CUDA(cudaEventRecord(e1, st));
    // statuses as the reference leaves them: OLD except the unexpanded level
    rc = table_fixup_status(t, pending, n_pending);
    if (rc) return rc;
    GX_CUDA(cudaMemcpyAsync(hc, ctr, sizeof(uint64_t) * CTR_N, cudaMemcpyDeviceToHost, st));
    GX_CUDA(cudaStreamSynchronize(st));
    float ms = 0;
    GX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    // occupancy counters of the table after the run
    unsigned long long cset[2] = {states, states - n_pending};
    GX_CUDA(cudaMemcpyAsync(ctr, cset, sizeof cset, cudaMemcpyHostToDevice, st));
    GX_CUDA(cudaStreamSynchronize(st));
    rep->states = states;
    rep->transitions = hc[LV_TRANS];
    rep->expanded = hc[LV_EXP];
    rep->iterations = rounds;
    rep->deadlocks_total = hc[LV_DL];
    rep->outcome = outcome;
    rep->deadlocks_kept = (int32_t)(kept.size() / v);
    if (deadlocks && !kept.empty()) memcpy(deadlocks, kept.data(), sizeof(uint32_t) * kept.size());
    rep->device_ms = ms;
    rep->probes = hc[LV_PROBES];
    rep->max_frontier = max_front;
    rep->kernels = gx_kernel_launches() - launches0;
    return GX_OK;
}

int gx_expand_route(gx_net* n, const gx_table* t, const uint32_t* d_front, uint64_t nfront,
                    int32_t ranks, uint32_t* d_out, uint64_t cap, uint64_t* d_counts,
                    uint64_t* d_offsets, uint64_t* transitions, uint64_t* deadlocks,
                    int32_t detect) {
    const uint32_t v = n->vlen;
    if (ranks < 1) {
        set_error("ranks must be >= 1");
        return GX_EINPUT;
    }
    cudaStream_t st = n->stream;
    if (ranks > 64) {
        set_error("at most 64 ranks");
        return GX_EINPUT;
    }
    // scratch: counters (8) + cursors (64) | flat successors (cap)
    const uint64_t head = 8 * 72;
    int rc = n->scratch.ensure(head + sizeof(uint32_t) * std::max<uint64_t>(cap, 1) * v);
    if (rc) return rc;
    unsigned long long* c = (unsigned long long*)n->scratch.p;
    uint32_t* flat = (uint32_t*)((char*)n->scratch.p + head);
    const uint64_t dl_cap = 1 << 16;
    rc = n->dl.ensure(sizeof(uint32_t) * dl_cap * v);
    if (rc) return rc;
    GX_CUDA(cudaMemsetAsync(c, 0, 64, st));
    unsigned long long h[8] = {0};
    if (nfront) {
        const int g = (int)std::min<uint64_t>((uint64_t)persistent_grid(), (nfront + 255) / 256);
        pick_flat((int)v)<<<g, 256, 0, st>>>(n->d, d_front, nfront, flat, cap, c, (uint32_t*)n->dl.p,
                                            dl_cap, detect);
        GX_LAUNCHED();
    }
    GX_CUDA(cudaMemcpyAsync(h, c, 64, cudaMemcpyDeviceToHost, st));
    GX_CUDA(cudaStreamSynchronize(st));
    if (h[3]) {
        set_error("successor buffer capacity (%llu vectors) exceeded", (unsigned long long)cap);
        return GX_EINTERNAL;
    }
    const uint64_t nsucc = h[0];
    GX_CUDA(cudaMemsetAsync(d_counts, 0, sizeof(uint64_t) * ranks, st));
    if (nsucc) {
        k_owner_hist<<<(int)((nsucc + 255) / 256), 256, 0, st>>>(t->d.salt, flat, nsucc, (int)v, ranks,
                                                                (unsigned long long*)d_counts);
        GX_LAUNCHED();
    }
    std::vector<unsigned long long> cnt(ranks), offs(ranks);
    GX_CUDA(cudaMemcpyAsync(cnt.data(), d_counts, sizeof(uint64_t) * ranks, cudaMemcpyDeviceToHost, st));
    GX_CUDA(cudaStreamSynchronize(st));
    unsigned long long acc = 0;
    for (int r = 0; r < ranks; r++) {
        offs[r] = acc;
        acc += cnt[r];
    }
    GX_CUDA(cudaMemcpyAsync(d_offsets, offs.data(), sizeof(uint64_t) * ranks, cudaMemcpyHostToDevice, st));
    if (nsucc) {
        unsigned long long* d_cur = c + 8;  // scatter cursors start at the offsets
        GX_CUDA(cudaMemcpyAsync(d_cur, offs.data(), sizeof(unsigned long long) * ranks,
                                cudaMemcpyHostToDevice, st));
        k_owner_scatter<<<(int)((nsucc + 255) / 256), 256, 0, st>>>(t->d.salt, flat, nsucc, (int)v, ranks,
                                                                   d_cur, d_out);
        GX_LAUNCHED();
        GX_CUDA(cudaStreamSynchronize(st));
    }
    if (transitions) *transitions = h[1];
    if (deadlocks) *deadlocks = h[2];
    n->dl_recorded = std::min<uint64_t>(h[2], dl_cap);
    if (h[2] > dl_cap) {
        // more deadlocks than records: the exact 100 smallest, left in dl
        std::vector<uint32_t> kept;
        rc = rescan_deadlocks(n, d_front, nfront, (uint32_t*)n->dl.p, dl_cap, c + 4, st, kept);
        if (rc) return rc;
        GX_CUDA(cudaMemcpyAsync(n->dl.p, kept.data(), sizeof(uint32_t) * kept.size(), cudaMemcpyHostToDevice, st));
        GX_CUDA(cudaStreamSynchronize(st));
        n->dl_recorded = kept.size() / v;
    }
    return GX_OK;
}

int gx_net_deadlocks(gx_net* n, uint32_t* out, uint64_t cap, uint64_t* count) {
    const uint64_t k = std::min<uint64_t>(n->dl_recorded, cap);
    if (count) *count = n->dl_recorded;
    if (out && k) {
        GX_CUDA(cudaMemcpyAsync(out, n->dl.p, sizeof(uint32_t) * k * n->vlen, cudaMemcpyDeviceToHost,
                                n->stream));
        GX_CUDA(cudaStreamSynchronize(n->stream));
    }
    return GX_OK;
}

int gx_insert_append(gx_table* t, const uint32_t* d_keys, uint64_t n, uint32_t* d_next, uint64_t cap,
                     uint64_t* n_next, int32_t* table_full) {
    append_kernel_t k = pick_append(t->d, 0);
    if (!k) {
        set_error("no append kernel for bw=%u vlen=%u", t->d.bw, t->d.vlen);
        return GX_EINPUT;
    }
    cudaStream_t st = t->stream;
    unsigned long long* c = (unsigned long long*)t->d_ctr + CTR_SCRATCH;  // cells 3..5
    GX_CUDA(cudaMemsetAsync(c, 0, 3 * sizeof(unsigned long long), st));
    if (n) {
        const int g = (int)std::min<uint64_t>((uint64_t)persistent_grid(), (n + 255) / 256 + 1);
        k<<<g, 256, 0, st>>>(t->d, d_keys, n, d_next, cap, c);
        GX_LAUNCHED();
    }
    unsigned long long h[3];
    GX_CUDA(cudaMemcpyAsync(h, c, sizeof h, cudaMemcpyDeviceToHost, st));
    GX_CUDA(cudaStreamSynchronize(st));
    if (h[2]) {
        set_error("next-frontier capacity (%llu vectors) exceeded", (unsigned long long)cap);
        return GX_EINTERNAL;
    }
    // keep occupancy in step
    unsigned long long occ[1];
    GX_CUDA(cudaMemcpyAsync(occ, t->d_ctr + CTR_OCCUPIED, 8, cudaMemcpyDeviceToHost, st));
    GX_CUDA(cudaStreamSynchronize(st));
    occ[0] += h[0];
    GX_CUDA(cudaMemcpyAsync(t->d_ctr + CTR_OCCUPIED, occ, 8, cudaMemcpyHostToDevice, st));
    if (n_next) *n_next = h[0];
    if (table_full) *table_full = h[1] ? 1 : 0;
    return GX_OK;
}

int gx_owner_of(const gx_table* t, const uint32_t* keys, uint64_t n, int32_t ranks, int32_t* owner) {
    if (n == 0) return GX_OK;
    const uint32_t v = t->d.vlen;
    uint32_t* dk = nullptr;
    int32_t* dout = nullptr;
    GX_CUDA(cudaMalloc(&dk, sizeof(uint32_t) * n * v));
    GX_CUDA(cudaMalloc(&dout, sizeof(int32_t) * n));
    GX_CUDA(cudaMemcpy(dk, keys, sizeof(uint32_t) * n * v, cudaMemcpyHostToDevice));
    k_owner_of<<<(int)((n + 255) / 256), 256>>>(t->d.salt, dk, n, (int)v, ranks, dout);
    GX_LAUNCHED();
    GX_CUDA(cudaMemcpy(owner, dout, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
    cudaFree(dk);
    cudaFree(dout);
    return GX_OK;
}

int gx_bench_find_or_put(gx_table* t, uint64_t total, uint64_t dup, uint64_t seed, int32_t key_bits,
                         int32_t group, double* ms, uint64_t* found, uint64_t* inserted,
                         uint64_t* full) {
    return gx_bench_find_or_put_rows(t, total, dup, 0, seed, key_bits, group, ms, found, inserted, full,
                                     nullptr);
}

int gx_bench_find_or_put_rows(gx_table* t, uint64_t total, uint64_t dup, uint64_t row_base,
                              uint64_t seed, int32_t key_bits, int32_t group, double* ms,
                              uint64_t* found, uint64_t* inserted, uint64_t* full, uint64_t* loads) {
    if (total == 0 || dup == 0 || dup > total || key_bits < 1 || key_bits > 32) {
        set_error("bad benchmark parameters");
        return GX_EINPUT;
    }
    const TableDesc& T = t->d;
    if (T.mode == MODE_MARK && key_bits > 31) {
        set_error("table in mark mode stores keys of at most 31 bits per word");
        return GX_EINPUT;
    }
    const uint64_t unique = total / dup;
    if (T.vlen == 1 && unique + row_base > (1ull << key_bits)) {
        set_error("%llu unique one-word keys do not fit in %d bits", (unsigned long long)unique, key_bits);
        return GX_EINPUT;
    }
    // group 0 (auto) on in-band tables: the staged probe of the level kernel
    BenchKernel BK = (T.mode == MODE_MARK && group == 0) ? pick_bench_staged(T)
                                                          : BenchKernel{pick_bench(T, group), 0};
    bench_kernel_t k = BK.fn;
    if (!k) {
        set_error("no benchmark kernel for bw=%u vlen=%u group=%d", T.bw, T.vlen, group);
        return GX_EINPUT;
    }
    cudaStream_t st = t->stream;
    unsigned long long* c = (unsigned long long*)t->d_ctr + CTR_SCRATCH;
    GX_CUDA(cudaMemsetAsync(c, 0, 3 * sizeof(unsigned long long), st));
    BenchArgs B;
    B.total = total;
    B.dup = dup;
    B.unique = unique;
    B.row_base = row_base;
    B.seed = seed;
    B.key_bits = key_bits;
    int pb = 1;
    while ((1ull << pb) < total) pb++;
    B.perm_bits_n = pb;
    B.ctr = c;
    cudaEvent_t e0, e1;
    GX_CUDA(cudaEventCreate(&e0));
    GX_CUDA(cudaEventCreate(&e1));
    GX_CUDA(cudaEventRecord(e0, st));
    if (BK.smem) GX_CUDA(cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              (int)BK.smem));
    int resident = 0;
    GX_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&resident, k, 256, BK.smem));
    k<<<sm_count() * std::max(resident, 1), 256, BK.smem, st>>>(T, B);
    GX_LAUNCHED();
    GX_CUDA(cudaEventRecord(e1, st));
    unsigned long long h[3];
    GX_CUDA(cudaMemcpyAsync(h, c, sizeof h, cudaMemcpyDeviceToHost, st));
    GX_CUDA(cudaStreamSynchronize(st));
    if (loads) *loads = BK.smem ? h[2] : 0;  // counted by the staged kernel only
    float f = 0;
    GX_CUDA(cudaEventElapsedTime(&f, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    // occupancy bookkeeping
    unsigned long long occ;
    GX_CUDA(cudaMemcpy(&occ, t->d_ctr + CTR_OCCUPIED, 8, cudaMemcpyDeviceToHost));
    occ += h[0];
    GX_CUDA(cudaMemcpy(t->d_ctr + CTR_OCCUPIED, &occ, 8, cudaMemcpyHostToDevice));
    if (ms) *ms = f;
    if (inserted) *inserted = h[0];
    if (full) *full = h[1];
    if (found) *found = total - h[0] - h[1];
    return GX_OK;
}

}  // extern "C"
