// gx_shard.cu -- hash-owner sharded exploration.
//
// One gx_shard per GPU (or, for tests on one GPU, several per device in
// one process).  Shard r owns the states with owner_of_mix(key_mix) == r and
// holds that part of the state table.  One BFS level is two kernels with a
// cross-GPU barrier between them:
//
//   A  k_level_routed  expand the local frontier, drop block-cache hits,
//                      store successors owned by peers straight into the
//                      peers' inboxes (P2P stores over NVLink into
//                      CUDA-IPC-mapped memory), FINDORPUT the locally
//                      owned ones and append the inserted to the next
//                      frontier -- the all-to-all is fused into the
//                      expansion; no NCCL payload exchange, no staging
//                      buffer
//   -- barrier (the driver's all_reduce of the level counters) --
//   B  k_absorb        FINDORPUT the keys peers sent, append the inserted
//                      to the same next frontier
//
// Levels stay global BFS levels, so iterations / levels / transitions are
// the single-GPU (and reference, explore.py:212-281) values.  The
// reference's only parallelism is a bucket-range split of one shared
// table between CPU workers (explore.py:284-286).
#include <algorithm>
#include <cstring>
#include <vector>

#include "gx_level.cuh"
#include "gx_part.cuh"
#include "gx_bench.cuh"

namespace gx {

#ifndef GX_ABSORB_CACHE
#define GX_ABSORB_CACHE 1  // the block-local dedup cache in front of the inbox probes too
#endif

template <int BW, int V>
__global__ void __launch_bounds__(256, GX_STAGED_MINB) k_level_routed(TableDesc T, NetDesc N, LevelArgs A, RouteArgs R,
                                                                      AbsorbArgs AB) {
    level_staged_body<BW, V, true>(T, N, A, R, AB);
}

// FINDORPUT the inbox (n = *count keys, clamped to cap); inserted keys go to
// the next frontier through the level's LevelArgs.
template <int BW, int V>
__global__ void __launch_bounds__(256, GX_STAGED_MINB) k_absorb(TableDesc T, LevelArgs A, const uint32_t* __restrict__ inbox,
                                                  const unsigned long long* count, uint64_t cap,
                                                  const unsigned long long* use_alt = nullptr,
                                                  const uint32_t* __restrict__ alt = nullptr,
                                                  const unsigned long long* alt_count = nullptr,
                                                  uint64_t alt_cap = 0) {
    // partitioned mode: when the duplicate filter's output overflowed
    // (*use_alt), absorb the unfiltered sub-partition instead
    if (use_alt && *use_alt) {
        inbox = alt;
        count = alt_count;
        cap = alt_cap;
    }
    using L = StagedSmem<BW, V>;
    using S = Staged<BW, V>;
    constexpr int QCAP = QWORDS / V;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    uint32_t* q = reinterpret_cast<uint32_t*>(smem) + wid * QWORDS;
    unsigned long long* sbkt = reinterpret_cast<unsigned long long*>(smem + L::Q) + wid * S::SB_STRIDE;
    uint4* stage = reinterpret_cast<uint4*>(smem + L::Q + L::B + (size_t)wid * S::STAGE_BYTES);
    staged_init(sbkt, S::KB);
    unsigned long long* dcache = reinterpret_cast<unsigned long long*>(smem + L::FIXED);
    const uint32_t cmask = (V <= 2 && GX_ABSORB_CACHE) ? A.cache_mask : 0u;
    if (cmask) {
        for (uint32_t i = threadIdx.x; i <= cmask; i += blockDim.x) dcache[i] = 0ull;
        __syncthreads();
    }
    const uint64_t sent = *count;
    if (sent > cap && blockIdx.x == 0 && threadIdx.x == 0) atomicExch(&A.ctr[LV_OVF], 1ull);
    const uint64_t n = min(sent, cap);
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    unsigned long long probes = 0;
    for (uint64_t base = warp * QCAP; base < n; base += nwarps * QCAP) {
        const uint32_t m0 = (uint32_t)min((uint64_t)QCAP, n - base);
        for (uint32_t x = lane; x < m0 * V; x += 32) q[x] = __ldcs(inbox + base * V + x);
        __syncwarp();
        uint32_t m = m0;
        if (cmask) m = cache_filter<V>(T, dcache, cmask, q, m);
        probes += lane == 0 ? m : 0;
        uint32_t full = 0;
        const uint32_t n_out = probe_staged<BW, V>(T, q, m, stage, sbkt, &full);
        if (__any_sync(FULLMASK, full != 0u) && lane == 0) atomicExch(&A.ctr[LV_FULL], 1ull);
        if (n_out) flush_out<V>(A, q, n_out);
        __syncwarp();
    }
    probes = warp_sum(probes);
    if (lane == 0 && probes) atomicAdd(&A.ctr[LV_PROBES], probes);
}

// ---- hash-partitioned FINDORPUT benchmark (multi-GPU configs[1]) ---------
// Positions [first, first + count) of the global duplication sequence
// (gx_bench.cuh): each warp generates QCAP keys, stores those owned by peers
// into their inboxes (route_remote, as the level kernel) and FINDORPUTs its
// own; the peers absorb their inboxes after the barrier (k_absorb).
// INSERTED results are counted through LevelArgs (out_limit 0: nothing is
// appended, LV_NEW counts).
template <int BW, int V>
__global__ void __launch_bounds__(256, GX_STAGED_MINB) k_bench_routed(TableDesc T, LevelArgs A, RouteArgs R,
                                                                      BenchArgs B, uint64_t first,
                                                                      uint64_t count) {
    using L = StagedSmem<BW, V>;
    using S = Staged<BW, V>;
    constexpr int QCAP = QWORDS / V;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    uint32_t* q = reinterpret_cast<uint32_t*>(smem) + wid * QWORDS;
    unsigned long long* sbkt = reinterpret_cast<unsigned long long*>(smem + L::Q) + wid * S::SB_STRIDE;
    uint4* stage = reinterpret_cast<uint4*>(smem + L::Q + L::B + (size_t)wid * S::STAGE_BYTES);
    staged_init(sbkt, S::KB);
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    unsigned long long* ovf = R.inbox_ctr[R.rank] + GX_PART_SUB_MAX;
    unsigned long long probes = 0, routed = 0;
    const uint64_t end = first + count;
    for (uint64_t base = first + warp * QCAP; base < end; base += nwarps * QCAP) {
        const uint32_t m = (uint32_t)min((uint64_t)QCAP, end - base);
        for (uint32_t k = lane; k < m; k += 32) {
            uint32_t key[V];
            bench_key<V>(B, base + k, key);
#pragma unroll
            for (int w = 0; w < V; w++) q[k * V + w] = key[w];
        }
        __syncwarp();
        const uint32_t mloc = route_remote<V>(T, R, q, m, ovf, &routed, reinterpret_cast<uint32_t*>(stage));
        probes += lane == 0 ? mloc : 0;
        uint32_t full = 0;
        const uint32_t n_out = probe_staged<BW, V>(T, q, mloc, stage, sbkt, &full);
        if (__any_sync(FULLMASK, full != 0u) && lane == 0) atomicExch(&A.ctr[LV_FULL], 1ull);
        if (n_out) flush_out<V>(A, q, n_out);
        __syncwarp();
    }
    probes = warp_sum(probes);
    routed = warp_sum(routed);
    __threadfence_system();
    if (lane == 0) {
        if (probes) atomicAdd(&A.ctr[LV_PROBES], probes);
        if (routed) atomicAdd(&A.ctr[LV_ROUTED], routed);
    }
}

typedef void (*bench_routed_t)(TableDesc, LevelArgs, RouteArgs, BenchArgs, uint64_t, uint64_t);

template <int BW>
static bench_routed_t pick_bench_routed_v(int v) {
    switch (v) {
        case 1: return k_bench_routed<BW, 1>;
        case 2: return k_bench_routed<BW, 2>;
        case 4: return k_bench_routed<BW, 4>;
    }
    return nullptr;
}

static bench_routed_t pick_bench_routed(const TableDesc& T) {
    switch (T.bw) {
        case 4: return pick_bench_routed_v<4>((int)T.vlen);
        case 8: return pick_bench_routed_v<8>((int)T.vlen);
        case 16: return pick_bench_routed_v<16>((int)T.vlen);
        case 32: return pick_bench_routed_v<32>((int)T.vlen);
    }
    return nullptr;
}

// ---- partitioned dedup mode (gx_part.cuh) ----------------------------
// K1: expand + route every successor into its partition (no table access)
template <int V>
__global__ void __launch_bounds__(256, 2) k_level_part(TableDesc T, NetDesc N, LevelArgs A, RouteArgs R,
                                                       PartArgs P) {
    level_part_body<V>(T, N, A, R, P);
}

// K2a: one sub-partition of this shard through the L2 duplicate filter:
// the first occurrence of each key in the chunk is appended (mark bit
// cleared) to uniq; k_absorb then FINDORPUTs uniq (K2b).  No shared
// memory, so many more warps keep set lookups in flight than the probe
// kernel could.  Keys arrive with the mark bit set.
template <int V>
__global__ void __launch_bounds__(256, 4) k_dedup(TableDesc T, const uint32_t* __restrict__ keys,
                                                  const unsigned long long* count, uint64_t cap, void* set,
                                                  uint32_t groups, uint32_t* uniq, unsigned long long* uniq_ctr,
                                                  uint64_t uniq_cap, unsigned long long* ovf) {
    constexpr int KPL = 4;  // keys per lane with their set lookups in flight
    const int lane = threadIdx.x & 31;
    const uint64_t n = min((uint64_t)*count, cap);
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    const uint32_t unmark = ~T.mark;
    for (uint64_t base = warp * (32 * KPL); base < n; base += nwarps * (32 * KPL)) {
        uint32_t km[KPL][V];
        bool first[KPL];
#pragma unroll
        for (int i = 0; i < KPL; i++) {
            const uint64_t e = base + i * 32 + lane;
            const bool a = e < n;
            if (a) {
                if (V == 2) {
                    const uint2 x = __ldcs(reinterpret_cast<const uint2*>(keys + e * 2));
                    km[i][0] = x.x;
                    km[i][1 % V] = x.y;
                } else if (V == 4) {
                    const uint4 x = __ldcs(reinterpret_cast<const uint4*>(keys + e * 4));
                    km[i][0] = x.x;
                    km[i][1 % V] = x.y;
                    km[i][2 % V] = x.z;
                    km[i][3 % V] = x.w;
                } else {
#pragma unroll
                    for (int w = 0; w < V; w++) km[i][w] = __ldcs(keys + e * V + w);
                }
            } else {
#pragma unroll
                for (int w = 0; w < V; w++) km[i][w] = 0u;
            }
            bool marked = false;  // a written slot carries the mark bit
#pragma unroll
            for (int w = 0; w < V; w++) marked |= (km[i][w] & (w == (int)T.mark_word ? T.mark : 0u)) != 0u;
            first[i] = a && marked;
        }
        dedup_batch<V, KPL>(set, groups, km, first);
        uint32_t msk[KPL], tot = 0;
#pragma unroll
        for (int i = 0; i < KPL; i++) {
            msk[i] = __ballot_sync(FULLMASK, first[i]);
            tot += __popc(msk[i]);
        }
        if (!tot) continue;
        unsigned long long pos = 0;
        if (lane == 0) pos = atomicAdd(uniq_ctr, (unsigned long long)tot);
        pos = __shfl_sync(FULLMASK, pos, 0);
        if (pos + tot > uniq_cap) {
            if (lane == 0) atomicExch(ovf, 1ull);
            continue;
        }
#pragma unroll
        for (int i = 0; i < KPL; i++) {
            if (first[i]) {
                uint32_t* d = uniq + (pos + __popc(msk[i] & lanemask_lt())) * V;
#pragma unroll
                for (int w = 0; w < V; w++) d[w] = w == (int)T.mark_word ? (km[i][w] & unmark) : km[i][w];
            }
            pos += __popc(msk[i]);
        }
    }
}

typedef void (*part_kernel_t)(TableDesc, NetDesc, LevelArgs, RouteArgs, PartArgs);
typedef void (*dedup_kernel_t)(TableDesc, const uint32_t*, const unsigned long long*, uint64_t, void*, uint32_t,
                               uint32_t*, unsigned long long*, uint64_t, unsigned long long*);
typedef void (*absorb2_kernel_t)(TableDesc, LevelArgs, const uint32_t*, const unsigned long long*, uint64_t,
                                 const unsigned long long*, const uint32_t*, const unsigned long long*, uint64_t);

struct PartKernels {
    part_kernel_t a;     // K1: expand + route
    dedup_kernel_t b;    // K2a: duplicate filter
    absorb2_kernel_t c;  // K2b: FINDORPUT of the first occurrences
    size_t smem_a, smem_c;
};

template <int BW>
static PartKernels pick_part_v(int v) {
    switch (v) {
        case 1: return {k_level_part<1>, k_dedup<1>, k_absorb<BW, 1>, PartSmem<1>::FIXED, StagedSmem<BW, 1>::FIXED};
        case 2: return {k_level_part<2>, k_dedup<2>, k_absorb<BW, 2>, PartSmem<2>::FIXED, StagedSmem<BW, 2>::FIXED};
        case 4: return {k_level_part<4>, k_dedup<4>, k_absorb<BW, 4>, PartSmem<4>::FIXED, StagedSmem<BW, 4>::FIXED};
    }
    return {nullptr, nullptr, nullptr, 0, 0};
}

static PartKernels pick_part(const TableDesc& T) {
    switch (T.bw) {
        case 4: return pick_part_v<4>((int)T.vlen);
        case 8: return pick_part_v<8>((int)T.vlen);
        case 16: return pick_part_v<16>((int)T.vlen);
        case 32: return pick_part_v<32>((int)T.vlen);
    }
    return {nullptr, nullptr, nullptr, 0, 0};
}

typedef void (*routed_kernel_t)(TableDesc, NetDesc, LevelArgs, RouteArgs, AbsorbArgs);
typedef void (*absorb_kernel_t)(TableDesc, LevelArgs, const uint32_t*, const unsigned long long*, uint64_t,
                                const unsigned long long*, const uint32_t*, const unsigned long long*, uint64_t);

struct ShardKernels {
    routed_kernel_t a;
    absorb_kernel_t b;
    size_t fixed_smem;  // dynamic shared memory besides the cache (both kernels)
};

template <int BW>
static ShardKernels pick_shard_v(int v) {
    switch (v) {
        case 1: return {k_level_routed<BW, 1>, k_absorb<BW, 1>, StagedSmem<BW, 1>::FIXED};
        case 2: return {k_level_routed<BW, 2>, k_absorb<BW, 2>, StagedSmem<BW, 2>::FIXED};
        case 4: return {k_level_routed<BW, 4>, k_absorb<BW, 4>, StagedSmem<BW, 4>::FIXED};
    }
    return {nullptr, nullptr, 0};
}

static ShardKernels pick_shard(const TableDesc& T) {
    switch (T.bw) {
        case 4: return pick_shard_v<4>((int)T.vlen);
        case 8: return pick_shard_v<8>((int)T.vlen);
        case 16: return pick_shard_v<16>((int)T.vlen);
        case 32: return pick_shard_v<32>((int)T.vlen);
    }
    return {nullptr, nullptr, 0};
}

// inbox head: the per-sub-partition cursors and the overflow cell
// (gx_part.cuh PART_HEAD), padded so the keys start 4 KB aligned
static constexpr size_t INBOX_HEAD = (PART_HEAD + 4095) & ~size_t(4095);

}  // namespace gx

using namespace gx;

struct gx_shard {
    gx_net* n;
    gx_table* t;
    int32_t rank, world;
    cudaStream_t stream;
    ShardKernels K;
    uint32_t cslots;
    size_t smem;
    // own inbox: [u64 counter | pad][keys]
    void* inbox_block = nullptr;
    uint64_t inbox_cap;
    std::vector<void*> opened;  // peer blocks mapped through CUDA IPC
    RouteArgs R;
    bool connected = false;
    // two-ended frontier buffer
    DevBuf fb, dl, gf;
    uint64_t C;
    uint64_t gslots = 0;  // GPU-wide dedup filter entries (0 = off)
    const uint32_t* F = nullptr;
    uint64_t nF = 0;
    int rev = 1;
    unsigned long long new_base = 0, dl_base = 0;
    uint64_t dl_cap = 1 << 16;
    uint64_t states = 0;
    const uint32_t* pending = nullptr;
    uint64_t n_pending = 0;
    LevelArgs A;
    std::vector<uint32_t> kept, dlhost;
    // CUDA-event pairs around each kernel of the current level (A and B of
    // every chunk), read once at the end of the level
    std::vector<cudaEvent_t> ev;
    size_t ev_used = 0;
    double level_ms = 0;
    int32_t detect = 0;
    bool level_open = false;  // LevelArgs of the current level are set
    // partitioned dedup mode (gx_shard_set_mode)
    bool dedup = false;
    PartKernels P{};
    uint32_t nsub = 1;
    uint64_t cap_sub = 0;
    DevBuf set;
    uint32_t set_groups = 0;
    DevBuf snap;  // level counters before the current chunk's expansion (rollback)
    DevBuf uniq;  // first occurrences of one sub-partition: [ctr, ovf, pad..256 B][keys]
    uint64_t uniq_cap = 0;
    size_t smem_a = 0;
    // pipelined mode (gx_shard_set_pipeline): two inbox halves per shard;
    // chunk c routes into half c & 1 and absorbs half (c - 1) & 1 in the
    // same launch
    bool pipelined = false;
    uint64_t half = 0;        // keys per inbox half
    uint32_t chunk_idx = 0;   // chunks expanded in the current level
    void* peer_block[GX_MAX_SHARDS] = {};
};

extern "C" {

int gx_shard_create(gx_net* n, gx_table* t, int32_t rank, int32_t world, uint64_t inbox_capacity,
                    uint64_t frontier_capacity, int32_t cache_slots, int32_t filter_log2,
                    gx_shard** out) {
    *out = nullptr;
    const TableDesc& T = t->d;
    if (world < 1 || world > GX_MAX_SHARDS || rank < 0 || rank >= world) {
        set_error("shard rank %d / world %d outside 1..%d", rank, world, GX_MAX_SHARDS);
        return GX_EINPUT;
    }
    if (T.vlen != n->vlen) {
        set_error("table vector length %u != network vector length %u", T.vlen, n->vlen);
        return GX_EINPUT;
    }
    if (T.mode != MODE_MARK) {
        set_error("sharded exploration needs an in-band (mark bit) table; this packing has no spare bit");
        return GX_EINPUT;
    }
    ShardKernels K = pick_shard(T);
    if (!K.a) {
        set_error("no sharded level kernel for bw=%u vlen=%u", T.bw, T.vlen);
        return GX_EINPUT;
    }
    gx_shard* s = new gx_shard();
    s->n = n;
    s->t = t;
    s->rank = rank;
    s->world = world;
    s->stream = t->stream;
    s->K = K;
    s->cslots = 0;
    if (cache_slots > 0 && T.vlen <= 2) {
        const size_t budget = STAGED_SMEM_BUDGET;
        const size_t room = budget > K.fixed_smem ? (budget - K.fixed_smem) / 8 : 0;
        const uint32_t c = (uint32_t)std::min<size_t>({(size_t)cache_slots, (size_t)GX_CACHE_MAX_SLOTS, room});
        s->cslots = c >= 32 ? c : 0;
    }
    s->smem = K.fixed_smem + 8 * (size_t)s->cslots;
    s->inbox_cap = std::max<uint64_t>(inbox_capacity, 1024);
    s->C = std::max<uint64_t>(frontier_capacity, 1024);
    memset(&s->R, 0, sizeof s->R);
    s->R.world = world;
    s->R.rank = rank;
    s->R.inbox_cap = s->inbox_cap;
    cudaError_t e = cudaMalloc(&s->inbox_block, INBOX_HEAD + sizeof(uint32_t) * s->inbox_cap * T.vlen);
    if (e != cudaSuccess) {
        set_error("inbox allocation (%llu keys) failed: %s", (unsigned long long)s->inbox_cap,
                  cudaGetErrorString(e));
        delete s;
        return GX_EINTERNAL;
    }
    int rc = s->fb.ensure(sizeof(uint32_t) * s->C * T.vlen);
    if (!rc) rc = s->dl.ensure(sizeof(uint32_t) * s->dl_cap * T.vlen);
    if (!rc && filter_log2 > 0 && T.vlen <= 2) {
        s->gslots = 1ull << std::min(filter_log2, 28);
        rc = s->gf.ensure(8 * s->gslots);
    }
    if (rc) {
        cudaFree(s->inbox_block);
        delete s;
        return rc;
    }
    GX_CUDA(cudaMemsetAsync(s->inbox_block, 0, INBOX_HEAD, s->stream));
    GX_CUDA(cudaFuncSetAttribute((const void*)K.a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem));
    GX_CUDA(cudaFuncSetAttribute((const void*)K.b, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem));
    *out = s;
    return GX_OK;
}

int gx_shard_destroy(gx_shard* s) {
    if (!s) return GX_OK;
    cudaStreamSynchronize(s->stream);
    for (void* p : s->opened) cudaIpcCloseMemHandle(p);
    cudaFree(s->inbox_block);
    s->fb.release();
    s->dl.release();
    s->gf.release();
    s->set.release();
    s->snap.release();
    s->uniq.release();
    for (cudaEvent_t e : s->ev) cudaEventDestroy(e);
    delete s;
    return GX_OK;
}

int gx_shard_ipc_handle(gx_shard* s, uint8_t* out) {
    cudaIpcMemHandle_t h;
    GX_CUDA(cudaIpcGetMemHandle(&h, s->inbox_block));
    static_assert(sizeof(h) <= GX_IPC_HANDLE_BYTES, "IPC handle size");
    memset(out, 0, GX_IPC_HANDLE_BYTES);
    memcpy(out, &h, sizeof h);
    return GX_OK;
}

static void set_peer(gx_shard* s, int r, void* block) {
    s->peer_block[r] = block;
    s->R.inbox_ctr[r] = (unsigned long long*)block;
    s->R.inbox[r] = (uint32_t*)((char*)block + INBOX_HEAD);
}

// RouteArgs for inbox half `parity` of every peer (pipelined mode)
static RouteArgs route_half(const gx_shard* s, uint32_t parity) {
    RouteArgs R = s->R;
    const uint32_t v = s->t->d.vlen;
    for (int r = 0; r < s->world; r++) {
        R.inbox_ctr[r] = (unsigned long long*)s->peer_block[r] + parity;
        R.inbox[r] = (uint32_t*)((char*)s->peer_block[r] + INBOX_HEAD) + (uint64_t)parity * s->half * v;
    }
    R.inbox_cap = s->half;
    return R;
}

int gx_shard_connect(gx_shard* s, const uint8_t* handles) {
    static const uint8_t zero[GX_IPC_HANDLE_BYTES] = {};
    for (int r = 0; r < s->world; r++) {
        if (r == s->rank) {
            set_peer(s, r, s->inbox_block);
            continue;
        }
        const uint8_t* hb = handles + (size_t)r * GX_IPC_HANDLE_BYTES;
        if (!memcmp(hb, zero, GX_IPC_HANDLE_BYTES)) continue;  // same-process peer: gx_shard_link
        cudaIpcMemHandle_t h;
        memcpy(&h, hb, sizeof h);
        void* p = nullptr;
        GX_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        s->opened.push_back(p);
        set_peer(s, r, p);
    }
    for (int r = 0; r < s->world; r++)
        if (!s->R.inbox[r]) {
            s->connected = false;
            return GX_OK;  // waiting for gx_shard_link of the same-process peers
        }
    s->connected = true;
    return GX_OK;
}

int gx_shard_link(gx_shard* s, const gx_shard* peer) {
    if (peer->world != s->world || peer->inbox_cap != s->inbox_cap) {
        set_error("link: peer shard has world %d / inbox %llu, this one %d / %llu", peer->world,
                  (unsigned long long)peer->inbox_cap, s->world, (unsigned long long)s->inbox_cap);
        return GX_EINPUT;
    }
    set_peer(s, peer->rank, peer->inbox_block);
    bool all = true;
    for (int r = 0; r < s->world; r++) all = all && s->R.inbox[r] != nullptr;
    s->connected = all;
    return GX_OK;
}

int gx_shard_connect_local(gx_shard* const* shards, int32_t world) {
    for (int i = 0; i < world; i++) {
        gx_shard* s = shards[i];
        if (s->world != world || s->rank != i) {
            set_error("connect_local: shard %d has rank %d / world %d", i, s->rank, s->world);
            return GX_EINPUT;
        }
        if (s->inbox_cap != shards[0]->inbox_cap) {
            set_error("connect_local: inbox capacities differ");
            return GX_EINPUT;
        }
        for (int r = 0; r < world; r++) set_peer(s, r, shards[r]->inbox_block);
        s->connected = true;
    }
    return GX_OK;
}

int gx_shard_begin(gx_shard* s, int32_t owns_initial, int32_t detect_deadlocks, int32_t* table_full) {
    if (!s->connected) {
        set_error("shard not connected to its peers");
        return GX_EINPUT;
    }
    gx_table* t = s->t;
    int rc = gx_table_clear(t);
    if (rc) return rc;
    GX_CUDA(cudaMemsetAsync(s->inbox_block, 0, INBOX_HEAD, s->stream));
    if (s->gslots) GX_CUDA(cudaMemsetAsync(s->gf.p, 0, 8 * s->gslots, s->stream));
    s->F = (const uint32_t*)s->fb.p;
    s->nF = 0;
    s->rev = 1;
    s->new_base = s->dl_base = 0;
    s->states = 0;
    s->pending = nullptr;
    s->n_pending = 0;
    s->kept.clear();
    s->level_ms = 0;
    s->detect = detect_deadlocks;
    s->level_open = false;
    s->ev_used = 0;
    s->chunk_idx = 0;
    *table_full = 0;
    if (owns_initial) {
        rc = t->codes.ensure(16);
        if (rc) return rc;
        rc = table_find_or_put_dev(t, s->n->d_initial, 1, (uint8_t*)t->codes.p, nullptr, 0, 0);
        if (rc) return rc;
        GX_CUDA(cudaMemcpyAsync(s->fb.p, s->n->d_initial, sizeof(uint32_t) * t->d.vlen,
                                cudaMemcpyDeviceToDevice, s->stream));
        uint8_t code0 = 0;
        GX_CUDA(cudaMemcpyAsync(&code0, t->codes.p, 1, cudaMemcpyDeviceToHost, s->stream));
        GX_CUDA(cudaStreamSynchronize(s->stream));
        if (code0 == TABLE_FULL) {
            *table_full = 1;
        } else {
            s->nF = 1;
            s->states = 1;
            s->pending = s->F;
            s->n_pending = 1;
        }
    }
    // the level counters restart from zero (the table clear zeroed them);
    // the cleared inbox head must be in place before any peer (another
    // process) reserves space in it after the caller's barrier
    GX_CUDA(cudaStreamSynchronize(s->stream));
    return GX_OK;
}

static cudaEvent_t next_event(gx_shard* s) {
    if (s->ev_used == s->ev.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
        s->ev.push_back(e);
    }
    return s->ev[s->ev_used++];
}

// Level arguments fixed for the whole level (its chunks append to the same
// next frontier); set by the first expand of a level.
static void level_args(gx_shard* s) {
    gx_table* t = s->t;
    LevelArgs& A = s->A;
    A.front = s->F;
    A.nfront = s->nF;
    A.out = (uint32_t*)s->fb.p;
    A.out_cap = s->C;
    A.out_limit = s->C - s->nF;
    A.out_rev = s->rev;
    A.detect = s->detect;
    A.ctr = (unsigned long long*)t->d_ctr;
    A.new_base = s->new_base;
    A.dl_base = s->dl_base;
    A.dl = (uint32_t*)s->dl.p;
    A.dl_cap = s->dl_cap;
    A.cache_mask = s->cslots ? s->cslots - 1 : 0;
    A.gfilter_mask = s->gslots ? (uint32_t)(s->gslots - 1) : 0;
    A.gfilter = (unsigned long long*)s->gf.p;
    s->level_open = true;
}

int gx_shard_set_mode(gx_shard* s, int32_t dedup, int32_t set_log2) {
    if (!dedup) {
        s->dedup = false;
        return GX_OK;
    }
    const TableDesc& T = s->t->d;
    PartKernels P = pick_part(T);
    if (!P.a) {
        set_error("no partitioned level kernels for bw=%u vlen=%u", T.bw, T.vlen);
        return GX_EINPUT;
    }
    if (set_log2 < 10 || set_log2 > 26) {
        set_error("dedup set of 2^%d groups outside 2^10..2^26", set_log2);
        return GX_EINPUT;
    }
    s->P = P;
    s->set_groups = 1u << set_log2;
    int rc = s->set.ensure(32ull * s->set_groups);
    if (!rc) rc = s->snap.ensure(sizeof(uint64_t) * CTR_N);
    if (rc) return rc;
    // the K1 queue cache (block-local, optional) rides after its fixed part
    s->smem_a = ((P.smem_a + 15) & ~size_t(15)) + 8 * (size_t)s->cslots;
    if (s->smem_a > STAGED_SMEM_BUDGET * GX_STAGED_MINB / 2) {  // keep 2 blocks per SM
        s->smem_a = (P.smem_a + 15) & ~size_t(15);
    }
    GX_CUDA(cudaFuncSetAttribute((const void*)P.a, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->smem_a));
    GX_CUDA(cudaFuncSetAttribute((const void*)P.c, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem_c));
    // first occurrences of a sub-partition: a quarter of the inbox (more
    // only below 4x duplication; then the unfiltered sub-partition is
    // absorbed instead, decided on the device)
    s->uniq_cap = std::max<uint64_t>(s->inbox_cap / 4, 1 << 16);
    rc = s->uniq.ensure(256 + sizeof(uint32_t) * T.vlen * s->uniq_cap);
    if (rc) return rc;
    s->dedup = true;
    s->nsub = 1;
    s->cap_sub = s->inbox_cap;
    return GX_OK;
}

int gx_shard_set_partitions(gx_shard* s, uint32_t nsub) {
    if (nsub < 1 || nsub > GX_PART_SUB_MAX || (nsub & (nsub - 1)) || (uint64_t)nsub * s->world > GX_PART_BINS_MAX) {
        set_error("%u sub-partitions x %d shards: need a power of two within %d per shard, %d bins", nsub,
                  s->world, GX_PART_SUB_MAX, GX_PART_BINS_MAX);
        return GX_EINPUT;
    }
    s->nsub = nsub;
    s->cap_sub = s->inbox_cap / nsub;
    return GX_OK;
}

int gx_shard_expand_range(gx_shard* s, uint64_t begin, uint64_t count) {
    gx_table* t = s->t;
    const uint32_t v = t->d.vlen;
    if (!s->level_open) level_args(s);
    if (begin > s->nF) begin = s->nF;
    if (count > s->nF - begin) count = s->nF - begin;
    LevelArgs A = s->A;
    A.front = s->F + begin * v;
    A.nfront = count;
    cudaEvent_t a0 = next_event(s), a1 = next_event(s);
    if (s->dedup) {
        // counters before this chunk: gx_shard_rollback restores them
        GX_CUDA(cudaMemcpyAsync(s->snap.p, t->d_ctr, sizeof(uint64_t) * CTR_N, cudaMemcpyDeviceToDevice,
                                s->stream));
        GX_CUDA(cudaEventRecord(a0, s->stream));
        if (count) {
            PartArgs P;
            P.nsub = s->nsub;
            P.sub_log2 = (uint32_t)__builtin_ctz(s->nsub);
            P.cap_sub = s->cap_sub;
            A.cache_mask = s->smem_a > ((s->P.smem_a + 15) & ~size_t(15)) && s->cslots ? s->cslots - 1 : 0;
            const uint64_t want = (count + 31) / 32;
            const int g = (int)std::min<uint64_t>((uint64_t)sm_count() * 2, (want + 7) / 8);
            s->P.a<<<g, 256, s->smem_a, s->stream>>>(t->d, s->n->d, A, s->R, P);
            GX_LAUNCHED();
        }
        GX_CUDA(cudaEventRecord(a1, s->stream));
        return GX_OK;
    }
    GX_CUDA(cudaEventRecord(a0, s->stream));
    if (s->pipelined) {
        // route into half c & 1, absorb what peers routed here in chunk c - 1
        const uint32_t p = s->chunk_idx & 1u;
        AbsorbArgs AB{nullptr, nullptr, 0};
        unsigned long long* own = (unsigned long long*)s->inbox_block;
        if (s->chunk_idx > 0)
            AB = AbsorbArgs{(const uint32_t*)((char*)s->inbox_block + INBOX_HEAD) + (uint64_t)(p ^ 1u) * s->half * v,
                            own + (p ^ 1u), s->half};
        const uint64_t want = std::max<uint64_t>((count + 31) / 32, 1);
        const int g = (int)std::min<uint64_t>((uint64_t)sm_count() * GX_STAGED_MINB,
                                              s->chunk_idx > 0 ? (uint64_t)sm_count() * GX_STAGED_MINB : (want + 7) / 8);
        s->K.a<<<g, 256, s->smem, s->stream>>>(t->d, s->n->d, A, route_half(s, p), AB);
        GX_LAUNCHED();
        if (s->chunk_idx > 0) GX_CUDA(cudaMemsetAsync(own + (p ^ 1u), 0, 8, s->stream));
        s->chunk_idx++;
    } else if (count) {
        const uint64_t want = (count + 31) / 32;
        const int g = (int)std::min<uint64_t>((uint64_t)sm_count() * GX_STAGED_MINB, (want + 7) / 8);
        s->K.a<<<g, 256, s->smem, s->stream>>>(t->d, s->n->d, A, s->R, AbsorbArgs{nullptr, nullptr, 0});
        GX_LAUNCHED();
    }
    GX_CUDA(cudaEventRecord(a1, s->stream));
    return GX_OK;
}

int gx_shard_set_pipeline(gx_shard* s, int32_t on) {
    if (on && s->dedup) {
        set_error("the pipelined mode is for the fused levels, not the partitioned one");
        return GX_EINPUT;
    }
    s->pipelined = on != 0;
    s->half = s->inbox_cap / 2;
    s->chunk_idx = 0;
    return GX_OK;
}

int gx_shard_expand(gx_shard* s) { return gx_shard_expand_range(s, 0, ~0ull); }

int gx_shard_frontier(const gx_shard* s, uint64_t* n) {
    *n = s->nF;
    return GX_OK;
}

int gx_shard_bench_route(gx_shard* s, uint64_t total, uint64_t dup, uint64_t seed, int32_t key_bits,
                         uint64_t first, uint64_t count) {
    gx_table* t = s->t;
    const TableDesc& T = t->d;
    if (total == 0 || dup == 0 || dup > total || key_bits < 1 || key_bits > 31 || first + count > total) {
        set_error("bad benchmark parameters (mark-bit tables store at most 31 key bits per word)");
        return GX_EINPUT;
    }
    bench_routed_t k = pick_bench_routed(T);
    if (!k) {
        set_error("no routed benchmark kernel for bw=%u vlen=%u", T.bw, T.vlen);
        return GX_EINPUT;
    }
    if (!s->connected) {
        set_error("shard not connected to its peers");
        return GX_EINPUT;
    }
    if (!s->level_open) level_args(s);
    s->A.out_limit = 0;  // count INSERTED (LV_NEW), append nothing
    s->A.cache_mask = 0;
    BenchArgs B;
    B.total = total;
    B.dup = dup;
    B.unique = total / dup;
    B.row_base = 0;
    B.seed = seed;
    B.key_bits = key_bits;
    int pb = 1;
    while ((1ull << pb) < total) pb++;
    B.perm_bits_n = pb;
    B.ctr = nullptr;
    GX_CUDA(cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->K.fixed_smem));
    cudaEvent_t a0 = next_event(s), a1 = next_event(s);
    GX_CUDA(cudaEventRecord(a0, s->stream));
    if (count) {
        // pipelined shards: route into half 0, which absorb_chunk then drains
        const RouteArgs R = s->pipelined ? route_half(s, 0) : s->R;
        if (s->pipelined) s->chunk_idx = 1;
        k<<<sm_count() * GX_STAGED_MINB, 256, s->K.fixed_smem, s->stream>>>(T, s->A, R, B, first, count);
        GX_LAUNCHED();
    }
    GX_CUDA(cudaEventRecord(a1, s->stream));
    return GX_OK;
}

int gx_shard_bench_result(gx_shard* s, uint64_t* out, double* ms) {
    gx_table* t = s->t;
    unsigned long long* hc = (unsigned long long*)t->h_ctr;
    uint64_t ovf = 0;
    GX_CUDA(cudaMemcpyAsync(&ovf, (char*)s->inbox_block + 8 * GX_PART_SUB_MAX, 8, cudaMemcpyDeviceToHost, s->stream));
    GX_CUDA(cudaMemcpyAsync(hc, t->d_ctr, sizeof(uint64_t) * CTR_N, cudaMemcpyDeviceToHost, s->stream));
    GX_CUDA(cudaStreamSynchronize(s->stream));
    double tot = 0;
    for (size_t i = 0; i + 1 < s->ev_used; i += 2) {
        float x = 0;
        GX_CUDA(cudaEventElapsedTime(&x, s->ev[i], s->ev[i + 1]));
        tot += x;
    }
    s->ev_used = 0;
    s->level_open = false;
    out[0] = hc[LV_NEW];     // INSERTED (fresh keys stored in this shard)
    out[1] = hc[LV_FULL];    // TABLE_FULL seen
    out[2] = hc[LV_PROBES];  // FINDORPUTs run on this shard
    out[3] = hc[LV_ROUTED];  // keys sent to peers
    out[4] = ovf;            // an inbox overflowed
    if (ms) *ms = tot;
    return GX_OK;
}

int gx_shard_chunk_status(gx_shard* s, uint64_t* out) {
    uint64_t ovf = 0;
    GX_CUDA(cudaMemcpyAsync(&ovf, (char*)s->inbox_block + 8 * GX_PART_SUB_MAX, 8, cudaMemcpyDeviceToHost,
                            s->stream));
    GX_CUDA(cudaMemcpyAsync(s->t->h_ctr, s->t->d_ctr, sizeof(uint64_t) * CTR_N, cudaMemcpyDeviceToHost,
                            s->stream));
    GX_CUDA(cudaStreamSynchronize(s->stream));
    out[0] = ovf;
    out[1] = s->t->h_ctr[LV_ROUTED];
    out[2] = s->t->h_ctr[LV_EXP];
    return GX_OK;
}

int gx_shard_rollback(gx_shard* s) {
    if (!s->dedup) {
        set_error("rollback needs the partitioned mode");
        return GX_EINPUT;
    }
    GX_CUDA(cudaMemcpyAsync(s->t->d_ctr, s->snap.p, sizeof(uint64_t) * CTR_N, cudaMemcpyDeviceToDevice,
                            s->stream));
    GX_CUDA(cudaMemsetAsync(s->inbox_block, 0, 8 * (GX_PART_SUB_MAX + 1), s->stream));
    return GX_OK;
}

int gx_shard_absorb_chunk(gx_shard* s) {
    gx_table* t = s->t;
    cudaStream_t st = s->stream;
    if (!s->level_open) level_args(s);
    if (s->dedup) {
        unsigned long long* cur = (unsigned long long*)s->inbox_block;
        const uint32_t* keys = (const uint32_t*)((char*)s->inbox_block + INBOX_HEAD);
        cudaEvent_t b0 = next_event(s), b1 = next_event(s);
        GX_CUDA(cudaEventRecord(b0, st));
        unsigned long long* uctr = (unsigned long long*)s->uniq.p;  // [0] count, [1] overflow
        uint32_t* ukeys = (uint32_t*)((char*)s->uniq.p + 256);
        LevelArgs A = s->A;
        A.cache_mask = 0;
        for (uint32_t sub = 0; sub < s->nsub; sub++) {
            const uint32_t* skeys = keys + (uint64_t)sub * s->cap_sub * t->d.vlen;
            GX_CUDA(cudaMemsetAsync(s->set.p, 0, 32ull * s->set_groups, st));
            GX_CUDA(cudaMemsetAsync(uctr, 0, 16, st));
            s->P.b<<<sm_count() * 4, 256, 0, st>>>(t->d, skeys, cur + sub, s->cap_sub, s->set.p, s->set_groups,
                                                   ukeys, uctr, s->uniq_cap, uctr + 1);
            GX_LAUNCHED();
            s->P.c<<<sm_count() * GX_STAGED_MINB, 256, s->P.smem_c, st>>>(t->d, A, ukeys, uctr, s->uniq_cap,
                                                                         uctr + 1, skeys, cur + sub, s->cap_sub);
            GX_LAUNCHED();
        }
        GX_CUDA(cudaEventRecord(b1, st));
        GX_CUDA(cudaMemsetAsync(s->inbox_block, 0, 8 * (GX_PART_SUB_MAX + 1), st));
        return GX_OK;
    }
    // asynchronous: the inbox fill is only known on the device (a
    // persistent grid exits at once when nothing arrived, and flags an
    // overflowing inbox in LV_OVF); the counter is reset in stream order
    cudaEvent_t b0 = next_event(s), b1 = next_event(s);
    GX_CUDA(cudaEventRecord(b0, st));
    if (s->pipelined) {
        // the last chunk's half (the level's final absorb)
        const uint32_t p = (s->chunk_idx + 1) & 1u;  // (chunk_idx - 1) & 1
        unsigned long long* own = (unsigned long long*)s->inbox_block + p;
        const uint32_t* keys = (const uint32_t*)((char*)s->inbox_block + INBOX_HEAD) + (uint64_t)p * s->half * t->d.vlen;
        s->K.b<<<sm_count() * GX_STAGED_MINB, 256, s->smem, st>>>(t->d, s->A, keys, own, s->half, nullptr, nullptr,
                                                                 nullptr, 0);
        GX_LAUNCHED();
        GX_CUDA(cudaEventRecord(b1, st));
        GX_CUDA(cudaMemsetAsync(own, 0, 8, st));
        return GX_OK;
    }
    s->K.b<<<sm_count() * GX_STAGED_MINB, 256, s->smem, st>>>(t->d, s->A, s->R.inbox[s->rank],
                                                             s->R.inbox_ctr[s->rank], s->inbox_cap, nullptr,
                                                             nullptr, nullptr, 0);
    GX_LAUNCHED();
    GX_CUDA(cudaEventRecord(b1, st));
    GX_CUDA(cudaMemsetAsync(s->R.inbox_ctr[s->rank], 0, 8, st));
    return GX_OK;
}

int gx_shard_end_level(gx_shard* s, uint64_t* stats) {
    gx_table* t = s->t;
    const uint32_t v = t->d.vlen;
    cudaStream_t st = s->stream;
    unsigned long long* hc = (unsigned long long*)t->h_ctr;
    GX_CUDA(cudaMemcpyAsync(hc, t->d_ctr, sizeof(uint64_t) * CTR_N, cudaMemcpyDeviceToHost, st));
    GX_CUDA(cudaStreamSynchronize(st));
    // device time of this shard's kernels (other shards' kernels may run
    // between them on a shared stream, so pairs are timed one by one)
    for (size_t i = 0; i + 1 < s->ev_used; i += 2) {
        float ms = 0;
        GX_CUDA(cudaEventElapsedTime(&ms, s->ev[i], s->ev[i + 1]));
        s->level_ms += ms;
    }
    s->ev_used = 0;
    const uint64_t claims = s->nF;
    const uint64_t nnew = hc[LV_NEW] - s->new_base;
    s->new_base = hc[LV_NEW];
    if (hc[LV_DL] > s->dl_base) {
        const uint64_t d = hc[LV_DL] - s->dl_base;
        if (d <= s->dl_cap) {
            s->dlhost.resize(d * v);
            GX_CUDA(cudaMemcpyAsync(s->dlhost.data(), s->dl.p, sizeof(uint32_t) * d * v, cudaMemcpyDeviceToHost, st));
            GX_CUDA(cudaStreamSynchronize(st));
            keep_smallest(s->n, s->kept, s->dlhost.data(), d);
        } else {  // overflowed record buffer: re-derive this level's deadlocks exactly
            int rc = rescan_deadlocks(s->n, s->F, s->nF, (uint32_t*)s->dl.p, s->dl_cap,
                                      (unsigned long long*)t->d_ctr + CTR_SCRATCH, st, s->kept);
            if (rc) return rc;
        }
        s->dl_base = hc[LV_DL];
    }
    s->states += nnew;
    const uint32_t* Fn = s->rev ? (const uint32_t*)s->fb.p + (s->C - nnew) * v : (const uint32_t*)s->fb.p;
    s->pending = Fn;
    s->n_pending = nnew;
    s->F = Fn;
    s->nF = nnew;
    s->rev ^= 1;
    s->level_open = false;
    s->chunk_idx = 0;
    // per-level claims / new, then cumulative counters
    stats[GX_SH_CLAIMS] = claims;
    stats[GX_SH_NEW] = nnew;
    stats[GX_SH_TRANSITIONS] = hc[LV_TRANS];
    stats[GX_SH_DEADLOCKS] = hc[LV_DL];
    stats[GX_SH_TABLE_FULL] = hc[LV_FULL] ? 1 : 0;
    stats[GX_SH_OVERFLOW] = hc[LV_OVF] ? 1 : 0;
    stats[GX_SH_ROUTED] = hc[LV_ROUTED];
    stats[GX_SH_PROBES] = hc[LV_PROBES];
    return GX_OK;
}

int gx_shard_absorb(gx_shard* s, uint64_t* stats) {
    int rc = gx_shard_absorb_chunk(s);
    return rc ? rc : gx_shard_end_level(s, stats);
}

int gx_shard_finish(gx_shard* s, gx_report* rep, uint32_t* deadlocks) {
    gx_table* t = s->t;
    const uint32_t v = t->d.vlen;
    int rc = table_fixup_status(t, s->pending, s->n_pending);
    if (rc) return rc;
    unsigned long long* hc = (unsigned long long*)t->h_ctr;
    GX_CUDA(cudaMemcpyAsync(hc, t->d_ctr, sizeof(uint64_t) * CTR_N, cudaMemcpyDeviceToHost, s->stream));
    GX_CUDA(cudaStreamSynchronize(s->stream));
    memset(rep, 0, sizeof *rep);
    rep->states = s->states;
    rep->transitions = hc[LV_TRANS];
    rep->expanded = hc[LV_EXP];
    rep->deadlocks_total = hc[LV_DL];
    rep->deadlocks_kept = (int32_t)(s->kept.size() / v);
    rep->level_ms = s->level_ms;
    rep->probes = hc[LV_PROBES];
    if (deadlocks && !s->kept.empty()) memcpy(deadlocks, s->kept.data(), sizeof(uint32_t) * s->kept.size());
    // occupancy counters of this shard's table after the run
    unsigned long long cset[2] = {s->states, s->states - s->n_pending};
    GX_CUDA(cudaMemcpyAsync(t->d_ctr, cset, sizeof cset, cudaMemcpyHostToDevice, s->stream));
    GX_CUDA(cudaStreamSynchronize(s->stream));
    return GX_OK;
}

}  // extern "C"
