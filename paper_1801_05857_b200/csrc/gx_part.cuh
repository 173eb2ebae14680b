// gx_part.cuh -- the partitioned level: expansion with successors
// partitioned by owner shard and hash sub-range (K1), then per partition an
// exact level-wide duplicate filter in an L2-resident set followed by
// FINDORPUT of the first occurrences only (K2).
//
// Why: in a BFS level every new state is generated once per predecessor in
// the level -- T/S times (token ring N=19: 12.7x; the per-level distinct
// successors are ~1 per new state, profiles/README.md "dedup study").  The
// block-local cache of the fused kernel removes ~8% of them; the random
// table probes of the rest are the level's DRAM cost.  Here each successor
// costs one streamed 8-byte write + read and an L2 hit (the set lives in
// L2: 1.2e11 CAS/s, 2.8e11 loads/s measured, profiles/ s2c) instead of a
// 128-byte DRAM probe (3e10/s), and only the distinct successors probe the
// table.  Reference semantics are unchanged: FINDORPUT is idempotent, so
// which copy of a key probes does not matter (hashtable.py:224-280), and
// transitions are counted at expansion (network.py:184-238).
#pragma once
#include "gx_level.cuh"

namespace gx {

#ifndef GX_PART_BINS_MAX
#define GX_PART_BINS_MAX 128  // owner shards x sub-partitions routed per chunk
#endif
#ifndef GX_PQWORDS
#define GX_PQWORDS 1024  // K1 per-warp successor queue (words)
#endif
constexpr int PQWORDS = GX_PQWORDS;
#ifndef GX_PART_SUB_MAX
#define GX_PART_SUB_MAX 256  // sub-partitions per shard
#endif

// inbox block of a shard: [cursor u64 x SUB_MAX][overflow u64][pad] then keys
constexpr size_t PART_HEAD = 8 * (GX_PART_SUB_MAX + 8);

// Partition of a key: owner shard o (the fused engine's owner_of_mix) and
// sub-partition s from the next bits of the same 32-bit mix.
__device__ __forceinline__ uint32_t part_bin(uint32_t x, int world, uint32_t nsub) {
    const uint64_t p = (uint64_t)x * (uint64_t)world;
    const uint32_t o = (uint32_t)(p >> 32);
    const uint32_t s = (uint32_t)(((uint64_t)(uint32_t)p * nsub) >> 32);
    return o * nsub + s;
}

struct PartArgs {
    uint32_t nsub;       // sub-partitions per shard this chunk (a power of two)
    uint32_t sub_log2;   // log2(nsub)
    uint64_t cap_sub;    // keys per sub-partition
};

// Route keys q[0, m) (V words each, no mark bit) into their partitions:
// per-warp counting sort by bin in shared memory, one reservation atomic
// per non-empty bin, then runs of consecutive keys stored to the owner's
// partition (a peer's over NVLink).  Keys are stored with the mark bit so
// an unwritten slot (0) is never mistaken for a key.  scratch: this warp's
// QCAP keys of sorted buffer + bins words.
template <int V>
__device__ __forceinline__ void route_partitioned(const TableDesc& T, const RouteArgs& R, const PartArgs& P,
                                                  const uint32_t* q, uint32_t m, uint32_t* sq,
                                                  uint16_t* sbin, uint32_t* bo, uint32_t* hist,
                                                  unsigned long long* base, unsigned long long* ovf,
                                                  unsigned long long* routed) {
    const int lane = threadIdx.x & 31;
    const uint32_t nbins = (uint32_t)R.world * P.nsub;
    for (uint32_t b = lane; b < nbins; b += 32) hist[b] = 0;
    __syncwarp();
    // pass 1: bin of every key, rank within its bin (one leader per group);
    // bo[e] = bin << 16 | offset within bin
    for (uint32_t r0 = 0; r0 < m; r0 += 32) {
        const uint32_t e = r0 + lane;
        uint32_t bin = 0xffffu;
        if (e < m) {
            uint32_t key[V];
#pragma unroll
            for (int w = 0; w < V; w++) key[w] = q[e * V + w];
            bin = part_bin(key_mix<V>(key), R.world, P.nsub);
        }
        const uint32_t grp = __match_any_sync(FULLMASK, bin);
        const int leader = __ffs(grp) - 1;
        uint32_t before = 0;
        if (lane == leader && bin != 0xffffu) before = hist[bin];
        before = __shfl_sync(FULLMASK, before, leader);
        __syncwarp();
        if (lane == leader && bin != 0xffffu) hist[bin] = before + __popc(grp);
        __syncwarp();
        if (e < m) bo[e] = bin << 16 | (before + __popc(grp & lanemask_lt()));
    }
    // reservations (independent atomics, one per non-empty bin) and the
    // exclusive scan of the bin counts (sorted positions in sq)
    uint32_t run = 0;
    for (uint32_t b0 = 0; b0 < nbins; b0 += 32) {
        const uint32_t b = b0 + lane;
        const uint32_t c = b < nbins ? hist[b] : 0u;
        unsigned long long g = 0;
        const uint32_t o = b >> P.sub_log2, sb = b & (P.nsub - 1);
        if (c) {
            g = atomicAdd(R.inbox_ctr[o] + sb, (unsigned long long)c);
            if (g + c > P.cap_sub) atomicExch(ovf, 1ull);
        }
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULLMASK, incl, o);
            if (lane >= o) incl += y;
        }
        __syncwarp();
        if (b < nbins) {
            const uint32_t start = run + incl - c;
            hist[b] = start;  // hist now holds the sorted start of bin b
            // base[b]: slot of sorted position 0 of bin b (mod 2^64: it may
            // lie below 0, only positions >= start are used; |value| < 2^62),
            // or 2^63 when the bin overflows its sub-partition
            base[b] = g + c > P.cap_sub ? (1ull << 63) : (unsigned long long)sb * P.cap_sub + g - start;
            (void)o;
        }
        run += __shfl_sync(FULLMASK, incl, 31);
    }
    if (lane == 0) *routed += m;
    __syncwarp();
    // pass 2: counting-sort scatter into sq (with the mark bit)
    for (uint32_t e = lane; e < m; e += 32) {
        const uint32_t x = bo[e];
        const uint32_t bin = x >> 16, pos = hist[bin] + (x & 0xffffu);
        sbin[pos] = (uint16_t)bin;
#pragma unroll
        for (int w = 0; w < V; w++) sq[pos * V + w] = q[e * V + w] | (w == (int)T.mark_word ? T.mark : 0u);
    }
    __syncwarp();
    // pass 3: consecutive sorted keys -> consecutive partition slots
    for (uint32_t e = lane; e < m; e += 32) {
        const uint32_t b = sbin[e];
        const unsigned long long bb = base[b];
        if (bb != (1ull << 63)) {
            uint32_t* dst = R.inbox[b >> P.sub_log2] + (bb + e) * V;
            if (V == 2) {
                *reinterpret_cast<uint2*>(dst) = make_uint2(sq[e * 2], sq[e * 2 + 1]);
            } else if (V == 4) {
                *reinterpret_cast<uint4*>(dst) = make_uint4(sq[e * 4], sq[e * 4 + 1], sq[e * 4 + 2], sq[e * 4 + 3]);
            } else {
#pragma unroll
                for (int w = 0; w < V; w++) dst[w] = sq[e * V + w];
            }
        }
    }
    __syncwarp();
}

// K1: expand frontier states, drop block-cache hits, route every successor
// (own ones included) into its partition.  No table access.
template <int V>
struct PartSmem {
    static constexpr size_t Q = 8ull * PQWORDS * 4;                // successor queues
    static constexpr size_t SQ = 8ull * PQWORDS * 4;               // sorted queues
    static constexpr size_t SB = 8ull * (PQWORDS / V) * 2;         // bin of each sorted key
    static constexpr size_t BO = 8ull * (PQWORDS / V) * 4;         // bin and rank of each key
    static constexpr size_t H = 8ull * GX_PART_BINS_MAX * 4;       // bin counts / starts
    static constexpr size_t BS = 8ull * GX_PART_BINS_MAX * 8;      // bin reservations
    static constexpr size_t FIXED = BS + Q + SQ + BO + H + SB;
};

template <int V>
__device__ __forceinline__ void level_part_body(const TableDesc& T, const NetDesc& N, const LevelArgs& A,
                                                const RouteArgs& R, const PartArgs& P) {
    using L = PartSmem<V>;
    constexpr int QCAP = PQWORDS / V;
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int wid = threadIdx.x >> 5;
    unsigned long long* bbase = reinterpret_cast<unsigned long long*>(smem) + wid * GX_PART_BINS_MAX;
    uint32_t* q = reinterpret_cast<uint32_t*>(smem + L::BS) + wid * PQWORDS;
    uint32_t* sq = reinterpret_cast<uint32_t*>(smem + L::BS + L::Q) + wid * PQWORDS;
    uint32_t* bo = reinterpret_cast<uint32_t*>(smem + L::BS + L::Q + L::SQ) + wid * (PQWORDS / V);
    uint32_t* hist = reinterpret_cast<uint32_t*>(smem + L::BS + L::Q + L::SQ + L::BO) + wid * GX_PART_BINS_MAX;
    uint16_t* sbin = reinterpret_cast<uint16_t*>(smem + L::BS + L::Q + L::SQ + L::BO + L::H) + wid * (PQWORDS / V);
    unsigned long long* dcache = reinterpret_cast<unsigned long long*>(smem + ((L::FIXED + 15) & ~size_t(15)));
    const uint32_t cmask = A.cache_mask;
    if (cmask) {
        for (uint32_t i = threadIdx.x; i <= cmask; i += blockDim.x) dcache[i] = 0ull;
        __syncthreads();
    }
    unsigned long long* ovf = R.inbox_ctr[R.rank] + GX_PART_SUB_MAX;  // own overflow cell
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    unsigned long long trans = 0, expanded = 0, routed = 0;
    for (uint64_t base = warp * 32; base < A.nfront; base += nwarps * 32) {
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
            if (cmask) m = cache_filter<V>(T, dcache, cmask, q, m);
            route_partitioned<V>(T, R, P, q, m, sq, sbin, bo, hist, bbase, ovf, &routed);
        }
    }
    trans = warp_sum(trans);
    expanded = warp_sum(expanded);
    routed = warp_sum(routed);
    __threadfence_system();  // peer partition stores visible before the level barrier
    if (lane == 0) {
        if (routed) atomicAdd(&A.ctr[LV_ROUTED], routed);
        if (trans) atomicAdd(&A.ctr[LV_TRANS], trans);
        if (expanded) atomicAdd(&A.ctr[LV_EXP], expanded);
    }
}

// ------------------------------------------------------ K2 dedup set
// Open addressing over 32-byte groups (4 slots of 8 bytes for V <= 2, 2
// of 16 bytes for V = 4) in a set sized to stay in L2.  A key is looked up
// with one load of its group; only when it is absent does an empty slot
// get a CAS.  Returns true for the first occurrence (the copy that must
// probe the table); a full group answers "first" (a redundant probe, never
// a lost state).
template <int V>
struct DedupSlot;

template <>
struct DedupSlot<1> {
    using W = unsigned long long;
    static constexpr int PER = 4;
    __device__ static W word(const uint32_t* km) { return (W)km[0]; }
};
template <>
struct DedupSlot<2> {
    using W = unsigned long long;
    static constexpr int PER = 4;
    __device__ static W word(const uint32_t* km) { return (W)km[0] | ((W)km[1] << 32); }
};
template <>
struct DedupSlot<4> {
    using W = unsigned __int128;
    static constexpr int PER = 2;
    __device__ static W word(const uint32_t* km) {
        return (W)km[0] | ((W)km[1] << 32) | ((W)km[2] << 64) | ((W)km[3] << 96);
    }
};

__device__ __forceinline__ uint32_t dedup_index(uint32_t x, uint32_t groups) {
    uint32_t y = (x ^ 0x5BD1E995u) * 0x9E3779B1u;
    y ^= y >> 15;
    y *= 0x2C1B3C6Du;
    y ^= y >> 12;
    return (uint32_t)(((uint64_t)y * groups) >> 32);
}

template <int V>
__device__ __forceinline__ bool dedup_first(void* set, uint32_t groups, const uint32_t* km) {
    using S = DedupSlot<V>;
    using W = typename S::W;
    const W k = S::word(km);
    uint32_t x[V];
#pragma unroll
    for (int w = 0; w < V; w++) x[w] = km[w];
    W* g = reinterpret_cast<W*>(set) + (uint64_t)dedup_index(key_mix<V>(x), groups) * S::PER;
    const uint4 a = __ldcg(reinterpret_cast<const uint4*>(g));
    const uint4 b = __ldcg(reinterpret_cast<const uint4*>(g) + 1);
    W cur[S::PER];
    if (V == 4) {
        cur[0] = (W)a.x | ((W)a.y << 32) | ((W)a.z << 64) | ((W)a.w << 96);
        cur[1] = (W)b.x | ((W)b.y << 32) | ((W)b.z << 64) | ((W)b.w << 96);
    } else {
        cur[0] = (W)a.x | ((W)a.y << 32);
        cur[1] = (W)a.z | ((W)a.w << 32);
        cur[2 % S::PER] = (W)b.x | ((W)b.y << 32);
        cur[3 % S::PER] = (W)b.z | ((W)b.w << 32);
    }
#pragma unroll
    for (int i = 0; i < S::PER; i++)
        if (cur[i] == k) return false;
#pragma unroll
    for (int i = 0; i < S::PER; i++) {
        if (cur[i] != (W)0) continue;
        const W old = atomicCAS(g + i, (W)0, k);
        if (old == (W)0) return true;   // installed: first occurrence
        if (old == k) return false;     // another copy won the race
    }
    return true;  // group full: probe (redundant at worst)
}

// dedup_first for KPL keys per lane with all their group loads in flight
// at once, then all needed CASes back to back, then the verdicts (a CAS
// lost to another key re-runs dedup_first for that key alone, out of
// line).  first[i] in: key i is live; out: it is the first occurrence.
template <int V>
__device__ __noinline__ bool dedup_retry(void* set, uint32_t groups, const uint32_t* km) {
    return dedup_first<V>(set, groups, km);
}

template <int V, int KPL>
__device__ __forceinline__ void dedup_batch(void* set, uint32_t groups, const uint32_t (&km)[KPL][V],
                                            bool (&first)[KPL]) {
    using S = DedupSlot<V>;
    using W = typename S::W;
    if constexpr (V == 4) {  // 128-bit slots: one key at a time
#pragma unroll
        for (int i = 0; i < KPL; i++)
            if (first[i]) first[i] = dedup_retry<V>(set, groups, km[i]);
        return;
    }
    const uint4* base = reinterpret_cast<const uint4*>(set);
    uint32_t gi[KPL];
    uint4 a[KPL], b[KPL];
#pragma unroll
    for (int i = 0; i < KPL; i++) {
        uint32_t x[V];
#pragma unroll
        for (int w = 0; w < V; w++) x[w] = km[i][w];
        gi[i] = dedup_index(key_mix<V>(x), groups);
        a[i] = b[i] = make_uint4(0, 0, 0, 0);
        if (first[i]) {
            a[i] = __ldcg(base + 2 * (uint64_t)gi[i]);
            b[i] = __ldcg(base + 2 * (uint64_t)gi[i] + 1);
        }
    }
    const uint32_t hi_w = V == 2 ? 1 : 0;
    int cand[KPL];
#pragma unroll
    for (int i = 0; i < KPL; i++) {
        const uint32_t k0 = km[i][0], k1 = V == 2 ? km[i][hi_w % V] : 0u;
        const bool s0 = a[i].x == k0 && a[i].y == k1, s1 = a[i].z == k0 && a[i].w == k1;
        const bool s2 = b[i].x == k0 && b[i].y == k1, s3 = b[i].z == k0 && b[i].w == k1;
        const bool e0 = (a[i].x | a[i].y) == 0u, e1 = (a[i].z | a[i].w) == 0u;
        const bool e2 = (b[i].x | b[i].y) == 0u, e3 = (b[i].z | b[i].w) == 0u;
        cand[i] = e0 ? 0 : e1 ? 1 : e2 ? 2 : e3 ? 3 : -1;
        if (s0 || s1 || s2 || s3) {
            first[i] = false;
            cand[i] = -1;
        }
        if (!first[i]) cand[i] = -1;
    }
    W old[KPL];
#pragma unroll
    for (int i = 0; i < KPL; i++) {
        old[i] = 0;
        if (cand[i] >= 0)
            old[i] = atomicCAS(reinterpret_cast<W*>(set) + 4 * (uint64_t)gi[i] + cand[i], (W)0, S::word(km[i]));
    }
#pragma unroll
    for (int i = 0; i < KPL; i++) {
        if (cand[i] < 0 || old[i] == (W)0) continue;  // decided / installed: first
        if (old[i] == S::word(km[i])) first[i] = false;
        else first[i] = dedup_retry<V>(set, groups, km[i]);  // lost the slot to another key
    }
}

}  // namespace gx
