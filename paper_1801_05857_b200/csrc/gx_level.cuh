// gx_level.cuh -- the pieces of one BFS level shared by the single-GPU
// explorer (gx_explore.cu) and the hash-owner sharded one (gx_shard.cu):
// level arguments and counters, frontier staging, the block-local dedup
// cache, owner routing and the staged level body (expand -> cache ->
// [route] -> FINDORPUT -> next frontier).  Reference: explore.py:147-281,
// network.py:184-238, hashtable.py:224-280.
#pragma once
#include "gx_expand.cuh"
#include "gx_staged.cuh"
#include "gx_internal.h"

namespace gx {

// level counters live in the table's counter block
enum { LV_NEW = 8, LV_TRANS = 9, LV_EXP = 10, LV_DL = 11, LV_FULL = 12, LV_OVF = 13, LV_PROBES = 14, LV_ROUTED = 15 };

struct LevelArgs {
    const uint32_t* front;
    uint64_t nfront;
    uint32_t* out;        // next frontier region base
    uint64_t out_cap;     // vectors in the two-ended frontier buffer
    uint64_t out_limit;   // max vectors F' may take (cap - |F|)
    int32_t out_rev;      // F' position p lives at out[rev ? cap-1-p : p]
    int32_t detect;
    unsigned long long* ctr;
    unsigned long long new_base, dl_base;
    uint32_t* dl;
    uint64_t dl_cap;
    uint32_t cache_mask;  // block-local dedup cache slots - 1 (0 = no cache)
    uint32_t gfilter_mask;  // GPU-wide dedup filter slots - 1 (0 = none)
    unsigned long long* gfilter;
};

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
    return v;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <int V>
__device__ __forceinline__ void load_state(const uint32_t* p, uint32_t* s) {
    if (V == 1) {
        s[0] = __ldcs(p);
    } else if (V == 2) {
        uint2 x = __ldcs(reinterpret_cast<const uint2*>(p));
        s[0] = x.x;
        s[1] = x.y;
    } else if (V == 4) {
        uint4 x = __ldcs(reinterpret_cast<const uint4*>(p));
        s[0] = x.x;
        s[1] = x.y;
        s[2] = x.z;
        s[3] = x.w;
    } else {
#pragma unroll
        for (int w = 0; w < V; w++) s[w] = __ldcs(p + w);
    }
}

template <int V>
__device__ __forceinline__ void store_state(uint32_t* p, const uint32_t* s) {
    if (V == 2) {
        *reinterpret_cast<uint2*>(p) = make_uint2(s[0], s[1]);
    } else if (V == 4) {
        *reinterpret_cast<uint4*>(p) = make_uint4(s[0], s[1], s[2], s[3]);
    } else {
#pragma unroll
        for (int w = 0; w < V; w++) p[w] = s[w];
    }
}

// words of shared memory per warp for the successor queue, and the same
// again for the queue of freshly inserted keys (next-frontier staging)
#ifndef GX_STAGED_MINB
#define GX_STAGED_MINB 3  // resident blocks per SM the staged kernels are built for (B200 sweep: 3 > 2)
#endif
// dynamic shared memory one block may take so that GX_STAGED_MINB fit per SM
constexpr size_t STAGED_SMEM_BUDGET = (228 * 1024) / GX_STAGED_MINB - 1024 - 1024;
#ifndef GX_QWORDS
#define GX_QWORDS 1024  // B200 sweep (ring16): 512 -> 1024 words cut level time 17%
#endif
constexpr int QWORDS = GX_QWORDS;      // staged kernels: per-warp successor queue (words)
constexpr int QWORDS_REG = 512;        // register-group kernel (static shared memory)

// Copy the warp's staged next-frontier keys to global memory with one
// atomic per flush (the counter is shared by the whole grid).
template <int V>
__device__ __forceinline__ void flush_out(const LevelArgs& A, const uint32_t* outq, uint32_t n_out) {
    const int lane = threadIdx.x & 31;
    unsigned long long pos0 = 0;
    if (lane == 0) pos0 = atomicAdd(&A.ctr[LV_NEW], (unsigned long long)n_out) - A.new_base;
    pos0 = __shfl_sync(FULLMASK, pos0, 0);
    if (pos0 + n_out > A.out_limit) {
        if (lane == 0) atomicExch(&A.ctr[LV_OVF], 1ull);
        return;
    }
    for (uint32_t x = lane; x < n_out; x += 32) {
        const unsigned long long p = pos0 + x;
        const uint64_t slot = A.out_rev ? A.out_cap - 1 - p : p;
        store_state<V>(A.out + slot * V, outq + (uint64_t)x * V);
    }
}

// Block-local dedup cache (GPUexplore's per-block cache; the
// reference's LocalCache, explore.py:91-144): a direct-mapped table of
// cmask + 1 slots (any count: the slot is the high half of mix x slots,
// so the cache takes whatever shared memory the resident blocks leave) of
// 64-bit packed keys (stored with the mark bit, so 0 = empty) in dynamic
// shared memory.  atomicExch installs a key and returns the previous
// occupant; only a key that was already there is dropped, because whoever
// installed it has FINDORPUT it (or will) in this launch.  A forgotten key
// just costs a global probe, so the cache never changes results.
template <int V>
__device__ __forceinline__ unsigned long long cache_word(const TableDesc& T, const uint32_t* key) {
    unsigned long long kv = 0;
#pragma unroll
    for (int w = 0; w < V; w++)
        kv |= (unsigned long long)(key[w] | (w == (int)T.mark_word ? T.mark : 0u)) << (32 * w);
    return kv;
}

// Drop the successors in q[0, m) the block has already probed; survivors are
// compacted to the front of q (stable).  Returns their number.
template <int V>
__device__ __forceinline__ uint32_t cache_filter(const TableDesc& T, unsigned long long* cache,
                                                 uint32_t cmask, uint32_t* q, uint32_t m) {
    const int lane = threadIdx.x & 31;
    uint32_t kept = 0;
    for (uint32_t r0 = 0; r0 < m; r0 += 32) {
        const uint32_t e = r0 + lane;
        const bool a = e < m;
        uint32_t key[V];
#pragma unroll
        for (int w = 0; w < V; w++) key[w] = a ? q[e * V + w] : 0u;
        bool keep = false;
        if (a) {
            const unsigned long long kv = cache_word<V>(T, key);
            keep = atomicExch(&cache[__umulhi(key_mix<V>(key), cmask + 1u)], kv) != kv;
        }
        const uint32_t km = __ballot_sync(FULLMASK, keep);
        __syncwarp();
        if (keep) {
            const uint32_t p = kept + __popc(km & lanemask_lt());
#pragma unroll
            for (int w = 0; w < V; w++) q[p * V + w] = key[w];
        }
        kept += __popc(km);
        __syncwarp();
    }
    return kept;
}

// GPU-wide dedup filter: the same exchange protocol as the block cache on a
// direct-mapped array small enough to stay in L2 (and inside the TLB's
// reach), so a successor generated again anywhere on the GPU -- the BFS
// "diamonds" of independent moves -- skips its random probe of the big
// table.  Keys are only dropped when the filter already held them, i.e.
// someone has FINDORPUT (or is FINDORPUTting) them.  The filter is cleared
// with the table, so it never outlives the keys it vouches for.
template <int V>
__device__ __forceinline__ uint32_t global_filter(const TableDesc& T, unsigned long long* gf,
                                                  uint32_t gmask, uint32_t* q, uint32_t m) {
    const int lane = threadIdx.x & 31;
    uint32_t kept = 0;
    for (uint32_t r0 = 0; r0 < m; r0 += 32) {
        const uint32_t e = r0 + lane;
        const bool a = e < m;
        uint32_t key[V];
#pragma unroll
        for (int w = 0; w < V; w++) key[w] = a ? q[e * V + w] : 0u;
        bool keep = false;
        if (a) {
            const unsigned long long kv = cache_word<V>(T, key);
            const uint32_t idx = (key_mix<V>(key) * 0x2545F491u) & gmask;
            keep = atomicExch(&gf[idx], kv) != kv;
        }
        const uint32_t km = __ballot_sync(FULLMASK, keep);
        __syncwarp();
        if (keep) {
            const uint32_t p = kept + __popc(km & lanemask_lt());
#pragma unroll
            for (int w = 0; w < V; w++) q[p * V + w] = key[w];
        }
        kept += __popc(km);
        __syncwarp();
    }
    return kept;
}

// ------------------------------------------------ hash-owner routing
// Multi-GPU: rank `rank` of `world` owns the keys whose
// owner_of_mix(key_mix(key)) is `rank`.  The level kernel routes every successor it
// does not own straight into the owner's inbox over NVLink (peer pointers
// from CUDA IPC; in one process, plain device pointers), reserving room
// with one atomicAdd on the owner's inbox counter per (warp, owner,
// chunk); successors it owns are probed locally right away.  The owners
// FINDORPUT their inboxes after the level barrier (k_absorb, gx_shard.cu).
#ifndef GX_MAX_SHARDS
#define GX_MAX_SHARDS 16
#endif

struct RouteArgs {
    uint32_t* inbox[GX_MAX_SHARDS];                 // peer r's inbox keys (V words each)
    unsigned long long* inbox_ctr[GX_MAX_SHARDS];   // peer r's inbox fill counter
    uint64_t inbox_cap;                             // keys per inbox
    int32_t world, rank;
};

// Send the keys of q[0, m) owned by other ranks to their inboxes; the
// locally owned ones are compacted (stably) to the front of q.  Returns
// their number; *routed counts keys sent (lane 0).  scratch: 64 u32 of
// per-warp shared memory (per-owner counts and cursors).  Lanes with the
// same owner find each other with one match.any per 32 keys; each group's
// lowest lane updates the owner's count / cursor (one writer per owner).
template <int V>
__device__ __forceinline__ uint32_t route_remote(const TableDesc& T, const RouteArgs& R, uint32_t* q,
                                                 uint32_t m, unsigned long long* ovf,
                                                 unsigned long long* routed, uint32_t* scratch) {
    const int lane = threadIdx.x & 31;
    const int world = R.world;
    // GX_ROUTE_ALL: own keys go through the own inbox too, so every probe
    // happens in the absorb kernel (a B200 experiment; off by default)
#ifdef GX_ROUTE_ALL
    const int self = -1;
#else
    const int self = R.rank;
#endif
    uint32_t* cnt = scratch;        // [GX_MAX_SHARDS]
    uint32_t* cur = scratch + 32;   // [GX_MAX_SHARDS]
    if (lane < GX_MAX_SHARDS) {
        cnt[lane] = 0;
        cur[lane] = 0;
    }
    __syncwarp();
    // pass 1: keys per owner
    for (uint32_t r0 = 0; r0 < m; r0 += 32) {
        const uint32_t e = r0 + lane;
        int o = -1;
        if (e < m) {
            uint32_t key[V];
#pragma unroll
            for (int w = 0; w < V; w++) key[w] = q[e * V + w];
            o = owner_of_mix(key_mix<V>(key), world);
        }
        const uint32_t grp = __match_any_sync(FULLMASK, o);
        if (o >= 0 && (grp & lanemask_lt()) == 0) cnt[o] += __popc(grp);
        __syncwarp();
    }
    // reserve room in every peer inbox at once (independent remote atomics)
    const uint32_t mine = lane < world ? cnt[lane] : 0u;
    unsigned long long base = 0;
    bool ok = true;
    if (lane < world && lane != self && mine) {
        base = atomicAdd(R.inbox_ctr[lane], (unsigned long long)mine);
        if (base + mine > R.inbox_cap) {
            ok = false;
            atomicExch(ovf, 1ull);
        }
    }
    const uint32_t sent = __reduce_add_sync(FULLMASK, lane != self ? mine : 0u);
    if (lane == 0) *routed += sent;
    // pass 2: scatter (peer stores, consecutive per owner) / compact local
    for (uint32_t r0 = 0; r0 < m; r0 += 32) {
        const uint32_t e = r0 + lane;
        int o = -1;
        uint32_t key[V];
#pragma unroll
        for (int w = 0; w < V; w++) key[w] = 0u;
        if (e < m) {
#pragma unroll
            for (int w = 0; w < V; w++) key[w] = q[e * V + w];
            o = owner_of_mix(key_mix<V>(key), world);
        }
        const uint32_t grp = __match_any_sync(FULLMASK, o);
        const uint32_t pos = (o >= 0 ? cur[o] : 0u) + __popc(grp & lanemask_lt());
        const int src = o < 0 ? 0 : o;
        const unsigned long long b_o = __shfl_sync(FULLMASK, base, src);
        const int ok_o = __shfl_sync(FULLMASK, ok ? 1 : 0, src);
        __syncwarp();
        if (o >= 0 && (grp & lanemask_lt()) == 0) cur[o] += __popc(grp);
        if (o >= 0 && o != self) {
            if (ok_o) {
                uint32_t* dst = R.inbox[o] + (b_o + pos) * (uint64_t)V;
#pragma unroll
                for (int w = 0; w < V; w++) dst[w] = key[w];
            }
        } else if (o == self) {
            // pos counts this rank's keys so far: a stable in-place compaction
#pragma unroll
            for (int w = 0; w < V; w++) q[pos * V + w] = key[w];
        }
        __syncwarp();
    }
    return self < 0 ? 0u : cur[self];
}

// Cache filter and owner routing of q[0, m) in two passes instead of
// three (cache_filter + route_remote): pass 1 computes each key's 32-bit
// mix once for its cache slot AND its owner, drops cache hits, compacts the
// kept keys stably to the front of q and counts keys per owner (match_any
// leaders); then one reservation atomic per (call, remote owner); pass 2
// stores remote keys to their owner's inbox (consecutive per owner) and
// compacts own keys again.  Returns the number of own keys; *routed
// (lane 0) counts keys sent.  scratch: 96 u32 of the warp's idle stage
// buffer.  Results are those of cache_filter + route_remote.
template <int V, bool ROUTE>
__device__ __forceinline__ uint32_t filter_route(const TableDesc& T, const RouteArgs& R, unsigned long long* cache,
                                                 uint32_t cmask, uint32_t* q, uint32_t m, unsigned long long* ovf,
                                                 unsigned long long* routed, uint32_t* scratch) {
    const int lane = threadIdx.x & 31;
    const int world = ROUTE ? R.world : 1;
    const int self = ROUTE ? R.rank : 0;
    uint32_t* cnt = scratch;   // [32] keys per owner
    uint32_t* cur = scratch + 32;  // [32] owner cursors (pass 2)
    if (ROUTE) {
        cnt[lane] = 0;
        cur[lane] = 0;
        __syncwarp();
    }
    uint32_t kept = 0;
    for (uint32_t r0 = 0; r0 < m; r0 += 32) {
        const uint32_t e = r0 + lane;
        const bool a = e < m;
        uint32_t key[V];
#pragma unroll
        for (int w = 0; w < V; w++) key[w] = a ? q[e * V + w] : 0u;
        bool keep = a;
        int o = -1;
        if (a) {
            const uint32_t x = key_mix<V>(key);
            if (cmask) {
                const unsigned long long kv = cache_word<V>(T, key);
                keep = atomicExch(&cache[__umulhi(x, cmask + 1u)], kv) != kv;  // any slot count
            }
            if (keep && ROUTE) o = owner_of_mix(x, world);
        }
        if (ROUTE) {
            const uint32_t grp = __match_any_sync(FULLMASK, o);
            if (o >= 0 && (grp & lanemask_lt()) == 0) cnt[o] += __popc(grp);
        }
        const uint32_t km = __ballot_sync(FULLMASK, keep);
        __syncwarp();
        if (keep) {
            const uint32_t p = kept + __popc(km & lanemask_lt());
#pragma unroll
            for (int w = 0; w < V; w++) q[p * V + w] = key[w];
        }
        kept += __popc(km);
        __syncwarp();
    }
    if (!ROUTE) return kept;
    // reserve room in every peer inbox at once (independent remote atomics)
    const uint32_t mine = lane < world ? cnt[lane] : 0u;
    unsigned long long base = 0;
    bool ok = true;
    if (lane < world && lane != self && mine) {
        base = atomicAdd(R.inbox_ctr[lane], (unsigned long long)mine);
        if (base + mine > R.inbox_cap) {
            ok = false;
            atomicExch(ovf, 1ull);
        }
    }
    const uint32_t sent = __reduce_add_sync(FULLMASK, lane != self ? mine : 0u);
    if (lane == 0) *routed += sent;
    // pass 2: scatter (peer stores, consecutive per owner) / compact local
    for (uint32_t r0 = 0; r0 < kept; r0 += 32) {
        const uint32_t e = r0 + lane;
        int o = -1;
        uint32_t key[V];
#pragma unroll
        for (int w = 0; w < V; w++) key[w] = 0u;
        if (e < kept) {
#pragma unroll
            for (int w = 0; w < V; w++) key[w] = q[e * V + w];
            o = owner_of_mix(key_mix<V>(key), world);
        }
        const uint32_t grp = __match_any_sync(FULLMASK, o);
        const uint32_t pos = (o >= 0 ? cur[o] : 0u) + __popc(grp & lanemask_lt());
        const int src = o < 0 ? 0 : o;
        const unsigned long long b_o = __shfl_sync(FULLMASK, base, src);
        const int ok_o = __shfl_sync(FULLMASK, ok ? 1 : 0, src);
        __syncwarp();
        if (o >= 0 && (grp & lanemask_lt()) == 0) cur[o] += __popc(grp);
        if (o >= 0 && o != self) {
            if (ok_o) {
                uint32_t* dst = R.inbox[o] + (b_o + pos) * (uint64_t)V;
                if (V == 2) {
                    *reinterpret_cast<uint2*>(dst) = make_uint2(key[0], key[1 % V]);
                } else {
#pragma unroll
                    for (int w = 0; w < V; w++) dst[w] = key[w];
                }
            }
        } else if (o == self) {
#pragma unroll
            for (int w = 0; w < V; w++) q[pos * V + w] = key[w];
        }
        __syncwarp();
    }
    return cur[self];
}

// The same level with the FINDORPUT of each successor chunk done by
// probe_staged (gx_staged.cuh): bucket loads staged in shared memory with
// cp.async, KB buckets in flight per warp.  All per-warp buffers live in
// dynamic shared memory: [q 8*QWORDS u32][bucket idx 8*KB u64]
// [stage 8*STAGE_BYTES][dedup cache].
#ifndef GX_OVERLAP
// 1: one-bucket-per-lane tables use level_overlap_body.  Exact (the GPU
// suite passes with it on) but slower on B200: ring19 1.53 vs 1.92, ring16
// 2.19 vs 2.81 ·10^9 states/s, peterson6 level 212 vs 152 ms
// (profiles/round2/s2zp_*; ring16 by slice size 64 / 128 / 256: 227 /
// 188 / 170 ms vs 142, s2zq_*): a round-sized slice of successors covers the
// ranges of about a third of the tile's states, so expand_state runs with
// a third of the lanes active several times per tile, and that issue cost
// outweighs the load latency it hides (other warps hid most of it already).
#define GX_OVERLAP 0
#endif

template <int BW, int V>
struct StagedSmem {
    using S = Staged<BW, V>;
    static constexpr size_t Q = 8ull * QWORDS * 4;
    static constexpr size_t B = 8ull * S::SB_STRIDE * 8;
    static constexpr size_t ST = 8ull * S::STAGE_BYTES;
    // per-warp routing scratch (64 u32) of the overlapped body, whose stage
    // buffer is busy while it routes
    static constexpr size_t SCR = GX_OVERLAP ? 8ull * 64 * 4 : 0;
    static constexpr size_t FIXED = Q + B + ST + SCR;
};

// Inbox keys to FINDORPUT in the same launch as the expansion (the
// sharded engine's pipelined mode): keys other shards routed here during
// the previous chunk.  keys == nullptr: none.
struct AbsorbArgs {
    const uint32_t* keys;
    const unsigned long long* count;
    uint64_t cap;
};

#ifndef GX_OV_CHUNK
#define GX_OV_CHUNK 128  // successors emitted per probe round
#endif

// The level body for tables whose warp stages one bucket per lane
// (probe_refill): the same work as level_staged_body, software-pipelined
// so that a warp's bucket loads overlap its own expansion.  Each turn of
// the loop (1) issues the cp.async bucket loads of the lanes' current
// keys, (2) while they fly, expands the next GX_OV_CHUNK successors of
// the warp's frontier tile (or loads the next tile) into the pending
// queue, filtered by the block cache and routed to their owners
// (filter_route), and (3) resolves the round exactly as probe_refill
// does -- FOUND / CAS claim / next hash function / TABLE_FULL -- and
// refills the lanes whose keys are done from the pending queue.  INSERTED
// keys collect in the queue's last quarter and go to the next frontier a
// flush at a time.  Each key's probe sequence and CAS protocol are those
// of hashtable.py:224-280, so the level's results are unchanged; only the
// interleaving differs.
template <int BW, int V, bool ROUTE>
__device__ __forceinline__ void level_overlap_body(const TableDesc& T, const NetDesc& N, const LevelArgs& A,
                                                   const RouteArgs& R) {
    using L = StagedSmem<BW, V>;
    using S = Staged<BW, V>;
    constexpr int CH = BW / 4, SPC = 4 / V;
    constexpr uint32_t QCAP = QWORDS / V;
    constexpr uint32_t OCAP = QCAP / 4;         // inserted keys awaiting a flush
    constexpr uint32_t PCAP = QCAP - OCAP;      // pending keys
    constexpr uint32_t CHUNK = GX_OV_CHUNK < PCAP / 2 ? GX_OV_CHUNK : PCAP / 2;
    constexpr unsigned long long SKIP = ~0ull;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    uint32_t* pq = reinterpret_cast<uint32_t*>(smem) + wid * QWORDS;
    uint32_t* oq = pq + PCAP * V;
    unsigned long long* sbkt = reinterpret_cast<unsigned long long*>(smem + L::Q) + wid * S::SB_STRIDE;
    uint4* stage = reinterpret_cast<uint4*>(smem + L::Q + L::B + (size_t)wid * S::STAGE_BYTES);
    uint32_t* scratch = reinterpret_cast<uint32_t*>(smem + L::Q + L::B + L::ST) + wid * 64;
    unsigned long long* dcache = reinterpret_cast<unsigned long long*>(smem + L::FIXED);
    const uint32_t cmask = V <= 2 ? A.cache_mask : 0u;
    if (cmask) {
        for (uint32_t i = threadIdx.x; i <= cmask; i += blockDim.x) dcache[i] = 0ull;
        __syncthreads();
    }
    const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    uint64_t base = ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5) * 32;  // next tile
    unsigned long long trans = 0, expanded = 0, probes = 0, routed = 0;
    const uint32_t mark_lo = T.mark;
    // the warp's frontier tile: this lane's state, its successor count n and
    // exclusive offset, the tile's total and how many are emitted
    uint32_t s[V];
    uint32_t n = 0, excl = 0, total = 0, c0 = 0;
    bool sh = false, tiles = true;
    // probe lane: key (with the mark), fold, hash function index
    uint32_t km[V];
    uint64_t h = 0;
    int r = 0;
    bool has = false;
    uint32_t ph = 0, pt = 0, n_out = 0;  // pending [ph, pt); inserted [0, n_out)
#pragma unroll
    for (int w = 0; w < V; w++) s[w] = km[w] = 0u;
    while (true) {
        // (1) this round's bucket loads
        const bool any = __any_sync(FULLMASK, has);
        const uint64_t bkt = has ? bucket_of(T, h, r) : 0;
        if (any) {
            sbkt[lane] = has ? bkt : SKIP;
            __syncwarp();
#pragma unroll
            for (int it = 0; it < CH; it++) {
                const uint32_t c = it * 32 + lane;
                const uint32_t k = c / CH, j = c % CH;
                const unsigned long long b = sbkt[k];
                if (b != SKIP) cp_async16(stage + k * CH + (j ^ (k & (CH - 1))), T.data + b * (uint64_t)BW + 4 * j);
            }
            cp_async_commit();
        }
        // (2) expansion while they fly
        if (c0 < total) {
            if (pt + CHUNK > PCAP && ph > 0) {  // slide the pending keys down
                const uint32_t nw = (pt - ph) * V;
                for (uint32_t x0 = 0; x0 < nw; x0 += 32) {
                    const uint32_t x = x0 + lane;
                    const uint32_t v = x < nw ? pq[ph * V + x] : 0u;
                    __syncwarp();
                    if (x < nw) pq[x] = v;
                    __syncwarp();
                }
                pt -= ph;
                ph = 0;
            }
            if (pt + CHUNK <= PCAP) {
                const uint32_t c1 = min(total, c0 + CHUNK);
                if (sh && n && excl < c1 && excl + n > c0) {
                    const uint32_t lo = max(c0, excl) - excl;
                    const uint32_t hi = min(c1, excl + n) - excl;
                    uint64_t dummy;
                    expand_state<V, true>(N, s, &dummy, lo, hi, pq + (uint64_t)(pt + excl + lo - c0) * V);
                }
                __syncwarp();
                uint32_t m = c1 - c0;
                if (ROUTE || cmask)
                    m = filter_route<V, ROUTE>(T, R, dcache, cmask, pq + pt * V, m, &A.ctr[LV_OVF], &routed,
                                               scratch);
                probes += lane == 0 ? m : 0u;
                pt += m;
                c0 = c1;
            }
        } else if (tiles) {
            int stop = 0;
            if (lane == 0)
                stop = (*(volatile unsigned long long*)&A.ctr[LV_FULL] != 0ull) ||
                       (*(volatile unsigned long long*)&A.ctr[LV_OVF] != 0ull);
            if (__shfl_sync(FULLMASK, stop, 0) || base >= A.nfront) {
                tiles = false;
                if (stop) ph = pt;  // abandon the level's remaining keys
            } else {
                const uint64_t idx = base + lane;
                sh = idx < A.nfront;
                if (sh)
                    load_state<V>(A.front + idx * V, s);
                n = 0;
                if (sh) {
                    uint64_t cnt = 0;
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
                total = __shfl_sync(FULLMASK, incl, 31);
                excl = incl - n;
                c0 = 0;
                base += nwarps * 32;
            }
        }
        // (3) resolve the round
        if (any) {
            cp_async_wait0();
            __syncwarp();
            int rc = -1, slot = -1;
            if (has) {
                for (int j = 0; j < CH && rc == -1; j++) {
                    const uint4 c4 = stage[lane * CH + (j ^ (lane & (CH - 1)))];
                    const uint32_t w4[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
                    for (int t = 0; t < SPC; t++) {
                        if (rc != -1) break;
                        bool zero = true, eq = true;
#pragma unroll
                        for (int w = 0; w < V; w++) {
                            zero = zero && w4[t * V + w] == 0u;
                            eq = eq && w4[t * V + w] == km[w];
                        }
                        if (eq) {
                            rc = FOUND;
                            slot = j * SPC + t;
                        } else if (zero) {
                            rc = -3;
                            slot = j * SPC + t;
                        }
                    }
                }
            }
            __syncwarp();
            if (rc == -3) {
                uint32_t old[V];
                SlotCas<V>::cas(T.data + bkt * (uint64_t)BW + slot * V, km, old);
                bool zero = true, eq = true;
#pragma unroll
                for (int w = 0; w < V; w++) {
                    zero = zero && old[w] == 0u;
                    eq = eq && old[w] == km[w];
                }
                if (zero) {
                    rc = INSERTED;
                } else if (eq) {
                    rc = FOUND;
                } else {
                    int64_t hd;
                    rc = resolve_lane_from<BW, V>(T, bkt, slot + 1, km, &hd);
                }
            }
            bool done = false;
            if (has) {
                if (rc == -1 && ++r >= (int)T.k) rc = TABLE_FULL;
                done = rc >= 0;
            }
            if (done && rc == TABLE_FULL) atomicExch(&A.ctr[LV_FULL], 1ull);
            const bool ins = done && rc == INSERTED;
            const uint32_t im = __ballot_sync(FULLMASK, ins);
            if (ins) {
                const uint32_t p = n_out + __popc(im & lanemask_lt());
#pragma unroll
                for (int w = 0; w < V; w++) oq[p * V + w] = km[w] & ~(w == (int)T.mark_word ? mark_lo : 0u);
            }
            n_out += __popc(im);
            has = has && !done;
            if (n_out + 32 > OCAP) {
                __syncwarp();
                flush_out<V>(A, oq, n_out);
                n_out = 0;
                __syncwarp();
            }
        }
        // refill the idle lanes from the pending keys
        const bool idle = !has;
        const uint32_t dm = __ballot_sync(FULLMASK, idle);
        if (idle) {
            const uint32_t idx = ph + __popc(dm & lanemask_lt());
            if (idx < pt) {
                uint32_t key[V];
#pragma unroll
                for (int w = 0; w < V; w++) key[w] = pq[idx * V + w];
                h = fold<V>(T.salt, key);
#pragma unroll
                for (int w = 0; w < V; w++) km[w] = key[w] | (w == (int)T.mark_word ? mark_lo : 0u);
                r = 0;
                has = true;
            }
        }
        ph = min(pt, ph + __popc(dm));
        __syncwarp();
        if (!tiles && c0 >= total && ph >= pt && !__any_sync(FULLMASK, has)) break;
    }
    if (n_out) flush_out<V>(A, oq, n_out);
    trans = warp_sum(trans);
    expanded = warp_sum(expanded);
    probes = warp_sum(probes);
    if (ROUTE) {
        __threadfence_system();  // peer inbox stores visible before the level barrier
    }
    if (lane == 0) {
        if (ROUTE && routed) atomicAdd(&A.ctr[LV_ROUTED], routed);
        if (trans) atomicAdd(&A.ctr[LV_TRANS], trans);
        if (expanded) atomicAdd(&A.ctr[LV_EXP], expanded);
        if (probes) atomicAdd(&A.ctr[LV_PROBES], probes);
    }
}

template <int BW, int V, bool ROUTE>
__device__ __forceinline__ void level_staged_body(const TableDesc& T, const NetDesc& N, const LevelArgs& A,
                                                  const RouteArgs& R, const AbsorbArgs AB = AbsorbArgs{nullptr, nullptr, 0}) {
    using L = StagedSmem<BW, V>;
    using S = Staged<BW, V>;
    constexpr int QCAP = QWORDS / V;
#if GX_OVERLAP && GX_REFILL && !GX_TMA
    if constexpr (S::KPL == 1) {
        if (!(V <= 2 && A.gfilter_mask) && !(ROUTE && AB.keys)) {
            level_overlap_body<BW, V, ROUTE>(T, N, A, R);
            return;
        }
    }
#endif
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    uint32_t* q = reinterpret_cast<uint32_t*>(smem) + wid * QWORDS;
    unsigned long long* sbkt = reinterpret_cast<unsigned long long*>(smem + L::Q) + wid * S::SB_STRIDE;
    uint4* stage = reinterpret_cast<uint4*>(smem + L::Q + L::B + (size_t)wid * S::STAGE_BYTES);
    unsigned long long* dcache = reinterpret_cast<unsigned long long*>(smem + L::FIXED);
    staged_init(sbkt, S::KB);
    const uint32_t cmask = V <= 2 ? A.cache_mask : 0u;
    if (cmask) {
        for (uint32_t i = threadIdx.x; i <= cmask; i += blockDim.x) dcache[i] = 0ull;
        __syncthreads();
    }
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    unsigned long long trans = 0, expanded = 0, probes = 0, routed = 0;
    // pipelined mode: every warp alternates a frontier tile with a batch of
    // inbox keys, so the pure-probe absorb work fills the latency gaps of
    // the expansion (one shard's table only: the TLB-friendly order holds)
    uint64_t n_abs = 0;
    if (ROUTE && AB.keys) n_abs = min((uint64_t)*AB.count, AB.cap);
    uint64_t batch = warp * QCAP;
    for (uint64_t base = warp * 32; base < A.nfront || batch < n_abs; base += nwarps * 32) {
        int stop = 0;
        if (lane == 0)
            stop = (*(volatile unsigned long long*)&A.ctr[LV_FULL] != 0ull) ||
                   (*(volatile unsigned long long*)&A.ctr[LV_OVF] != 0ull);
        if (__shfl_sync(FULLMASK, stop, 0)) break;
        if (ROUTE && batch < n_abs) {
            const uint32_t m0 = (uint32_t)min((uint64_t)QCAP, n_abs - batch);
            for (uint32_t x = lane; x < m0 * V; x += 32) q[x] = __ldcs(AB.keys + batch * V + x);
            __syncwarp();
            uint32_t m = m0;
            if (cmask)
                m = filter_route<V, false>(T, R, dcache, cmask, q, m, &A.ctr[LV_OVF], &routed,
                                           reinterpret_cast<uint32_t*>(stage));
            probes += lane == 0 ? m : 0;
            uint32_t full = 0;
            const uint32_t n_out = probe_staged<BW, V>(T, q, m, stage, sbkt, &full);
            if (__any_sync(FULLMASK, full != 0u) && lane == 0) atomicExch(&A.ctr[LV_FULL], 1ull);
            if (n_out) flush_out<V>(A, q, n_out);
            __syncwarp();
            batch += nwarps * QCAP;
        }
        if (base >= A.nfront) continue;
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
            if (V <= 2 && A.gfilter_mask) {  // the GPU-wide filter (off by default): the separate passes
                if (cmask) m = cache_filter<V>(T, dcache, cmask, q, m);
                m = global_filter<V>(T, A.gfilter, A.gfilter_mask, q, m);
                if (ROUTE)
                    m = route_remote<V>(T, R, q, m, &A.ctr[LV_OVF], &routed, reinterpret_cast<uint32_t*>(stage));
            } else if (ROUTE || cmask) {
                m = filter_route<V, ROUTE>(T, R, dcache, cmask, q, m, &A.ctr[LV_OVF], &routed,
                                           reinterpret_cast<uint32_t*>(stage));  // stage is idle here
            }
            probes += lane == 0 ? m : 0;
            uint32_t full = 0;
            const uint32_t n_out = probe_staged<BW, V>(T, q, m, stage, sbkt, &full);
            if (__any_sync(FULLMASK, full != 0u) && lane == 0) atomicExch(&A.ctr[LV_FULL], 1ull);
            if (n_out) flush_out<V>(A, q, n_out);
            __syncwarp();
        }
    }
    trans = warp_sum(trans);
    expanded = warp_sum(expanded);
    probes = warp_sum(probes);
    if (ROUTE) {
        routed = warp_sum(routed);
        __threadfence_system();  // peer inbox stores visible before the level barrier
    }
    if (lane == 0) {
        if (ROUTE && routed) atomicAdd(&A.ctr[LV_ROUTED], routed);
        if (trans) atomicAdd(&A.ctr[LV_TRANS], trans);
        if (expanded) atomicAdd(&A.ctr[LV_EXP], expanded);
        if (probes) atomicAdd(&A.ctr[LV_PROBES], probes);
    }
}

}  // namespace gx
