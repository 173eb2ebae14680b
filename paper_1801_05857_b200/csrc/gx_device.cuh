// gx_device.cuh -- device-side building blocks of the B200 state table.
//
// Table layout in HBM:
//   data   : u32[num_buckets * bw], bucket b at byte offset 4*bw*b.  Slot j
//            of a bucket sits at word offsets[j] (hashtable.py:161-171);
//            handle = b * spb + j (hashtable.py:260,274).
//   status : u8[num_buckets * stride], stride = (spb + 7) & ~7
//            (hashtable.py:174), EMPTY/CLAIMED/NEW/OLD per slot.
//
// Two insertion protocols:
//   MODE_MARK   a bit that no key sets (spare high bit of the packing
//               scheme) is set in every stored slot, so "slot == 0" means
//               EMPTY and a single 32/64/128-bit atomicCAS inserts a key.
//               The probe touches only the bucket's data sector(s).  Used
//               for vlen in {1,2,4} with contiguous slots.
//   MODE_STATUS the reference's claim -> write -> publish on the status byte
//               (hashtable.py:252-267), any vlen, any key bits.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define GX_MAXK 64
#define GX_MAXV 16
#define FULLMASK 0xffffffffu

namespace gx {

enum : uint32_t { EMPTY = 0, CLAIMED = 1, NEW = 2, OLD = 3 };
enum : int { FOUND = 0, INSERTED = 1, TABLE_FULL = 2 };
enum : uint32_t { MODE_MARK = 0, MODE_STATUS = 1 };

struct TableDesc {
    uint32_t* data;
    uint8_t* status;
    uint64_t nb;        // buckets
    uint64_t nb_magic;  // floor(2^64 / nb) (0 when nb == 1)
    uint32_t bw, vlen, spb, stride;
    uint32_t k, mode;
    uint32_t mark_word, mark;  // MODE_MARK: stored slot = key | (mark in word mark_word)
    uint32_t track_status;     // MODE_MARK: write NEW into status on insert
    uint32_t pad0;
    uint64_t salt;
    uint8_t offsets[32];
    uint64_t a[GX_MAXK];
    uint64_t b[GX_MAXK];
};

// fold, hashtable.py:205-211
template <int V>
__device__ __forceinline__ uint64_t fold(uint64_t salt, const uint32_t* p) {
    uint64_t h = salt;
#pragma unroll
    for (int i = 0; i < V; i++) {
        h = (h ^ (uint64_t)p[i]) * 0x9E3779B97F4A7C15ull;
        h ^= h >> 29;
    }
    return h;
}

__device__ __forceinline__ uint64_t fold_rt(uint64_t salt, const uint32_t* p, int v) {
    uint64_t h = salt;
    for (int i = 0; i < v; i++) {
        h = (h ^ (uint64_t)p[i]) * 0x9E3779B97F4A7C15ull;
        h ^= h >> 29;
    }
    return h;
}

// x mod d exactly, with m = floor(2^64 / d): q = mulhi(x, m) is floor(x/d)
// or one less, so one correction suffices (hashtable.py:217 semantics).
__device__ __forceinline__ uint64_t fastmod(uint64_t x, uint64_t d, uint64_t m) {
    if (m == 0) return 0;  // d == 1
    uint64_t q = __umul64hi(x, m);
    uint64_t r = x - q * d;
    return r >= d ? r - d : r;
}

// bucket_index, hashtable.py:213-217
__device__ __forceinline__ uint64_t bucket_of(const TableDesc& T, uint64_t h, int i) {
    return fastmod(T.a[i] * h + T.b[i], T.nb, T.nb_magic);
}

// A cheap 32-bit mix of a key (murmur3-style finaliser over its words): the
// owner rank of hash-owner sharding and the dedup caches' slot index.  Not
// the table hash (fold), so owners are decorrelated from bucket indices,
// and four times cheaper than fold + a 64-bit finaliser.
template <int V>
__device__ __forceinline__ uint32_t key_mix(const uint32_t* key) {
    uint32_t x = 0x9E3779B9u;
#pragma unroll
    for (int w = 0; w < V; w++) {
        x = (x ^ key[w]) * 0x85EBCA77u;
        x ^= x >> 13;
    }
    x *= 0xC2B2AE35u;
    return x ^ (x >> 16);
}

__device__ __forceinline__ uint32_t key_mix_rt(const uint32_t* key, int v) {
    uint32_t x = 0x9E3779B9u;
    for (int w = 0; w < v; w++) {
        x = (x ^ key[w]) * 0x85EBCA77u;
        x ^= x >> 13;
    }
    x *= 0xC2B2AE35u;
    return x ^ (x >> 16);
}

// owner rank in [0, ranks) of a key whose mix is x
__device__ __forceinline__ int owner_of_mix(uint32_t x, int ranks) {
    return (int)(((uint64_t)x * (uint64_t)ranks) >> 32);
}

__device__ __forceinline__ uint4 ldcg4(const uint32_t* p) {
    return __ldcg(reinterpret_cast<const uint4*>(p));
}

// ---------------------------------------------------------- slot CAS
template <int V>
struct SlotCas;

template <>
struct SlotCas<1> {
    // returns true on success; `old` gets the previous contents
    __device__ static bool cas(uint32_t* slot, const uint32_t* val, uint32_t* old) {
        uint32_t o = atomicCAS(slot, 0u, val[0]);
        old[0] = o;
        return o == 0u;
    }
};
template <>
struct SlotCas<2> {
    __device__ static bool cas(uint32_t* slot, const uint32_t* val, uint32_t* old) {
        unsigned long long v = (unsigned long long)val[0] | ((unsigned long long)val[1] << 32);
        unsigned long long o = atomicCAS(reinterpret_cast<unsigned long long*>(slot), 0ull, v);
        old[0] = (uint32_t)o;
        old[1] = (uint32_t)(o >> 32);
        return o == 0ull;
    }
};
template <>
struct SlotCas<4> {
    __device__ static bool cas(uint32_t* slot, const uint32_t* val, uint32_t* old) {
        unsigned __int128 v = (unsigned __int128)val[0] | ((unsigned __int128)val[1] << 32) |
                              ((unsigned __int128)val[2] << 64) | ((unsigned __int128)val[3] << 96);
        unsigned __int128 z = 0;
        unsigned __int128 o = atomicCAS(reinterpret_cast<unsigned __int128*>(slot), z, v);
        old[0] = (uint32_t)o;
        old[1] = (uint32_t)(o >> 32);
        old[2] = (uint32_t)(o >> 64);
        old[3] = (uint32_t)(o >> 96);
        return o == z;
    }
};

// ---------------------------------------------- MODE_MARK group probe
//
// G lanes (an aligned group inside the warp) cooperate on one key: each
// lane loads BW/4/G 16-byte chunks of the bucket (chunk c = gl + j*G, so
// for every j the group's loads are one contiguous segment), tests its
// slots for EMPTY (mark bit clear) and equality, and the masks are OR-ed
// over the group with xor shuffles.  The group leader then performs the
// claim: CAS into the first EMPTY slot; on a lost CAS it re-judges that
// slot against the winner's value and moves to the next slot it saw
// EMPTY (occupied slots are a bucket prefix and never change, so stale
// views only cost a failed CAS).  Bucket full -> next hash function.
//
// All 32 lanes must call this together (warp-uniform control); `active`
// marks lanes whose group carries a key.  Returns the code in every lane
// of the group; *handle is valid in every lane of the group.
template <int BW, int V, int G>
__device__ __forceinline__ int probe_mark(const TableDesc& T, bool active, const uint32_t* key,
                                          uint64_t h, int64_t* handle, int i0 = 0) {
    constexpr int CH = BW / 4;       // 16B chunks per bucket
    constexpr int CPL = CH / G;      // chunks per lane
    constexpr int SPC = 4 / V;       // slots per chunk
    static_assert(CH % G == 0, "group size must divide the bucket chunks");
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    const int leader = lane & ~(G - 1);

    uint32_t km[V];
#pragma unroll
    for (int w = 0; w < V; w++) km[w] = key[w] | (w == (int)T.mark_word ? T.mark : 0u);

    int code = -1;  // unresolved
    int64_t hd = -1;
    for (int i = i0; i < (int)T.k; i++) {
        bool todo = active && code < 0;
        if (!__any_sync(FULLMASK, todo)) break;
        uint32_t occ = 0, match = 0;
        uint64_t bucket = 0;
        if (todo) {
            bucket = bucket_of(T, h, i);
            const uint32_t* base = T.data + bucket * (uint64_t)BW;
            uint4 ch[CPL];
#pragma unroll
            for (int j = 0; j < CPL; j++) ch[j] = ldcg4(base + 4 * (gl + j * G));
#pragma unroll
            for (int j = 0; j < CPL; j++) {
                const uint32_t w4[4] = {ch[j].x, ch[j].y, ch[j].z, ch[j].w};
                const int c = gl + j * G;
#pragma unroll
                for (int t = 0; t < SPC; t++) {
                    const int s = c * SPC + t;
                    uint32_t ob = 0;
#pragma unroll
                    for (int w = 0; w < V; w++) ob |= w4[t * V + w] & (w == (int)T.mark_word ? T.mark : 0u);
                    bool o = ob != 0u;
                    bool m = true;
#pragma unroll
                    for (int w = 0; w < V; w++) m = m && (w4[t * V + w] == km[w]);
                    occ |= (o ? 1u : 0u) << s;
                    match |= (m ? 1u : 0u) << s;
                }
            }
        }
#pragma unroll
        for (int o = 1; o < G; o <<= 1) {
            occ |= __shfl_xor_sync(FULLMASK, occ, o);
            match |= __shfl_xor_sync(FULLMASK, match, o);
        }
        int rc = -1;
        int64_t rh = -1;
        if (todo && gl == 0) {
            constexpr uint32_t ALL = (BW / V) >= 32 ? 0xffffffffu : ((1u << (BW / V)) - 1u);
            if (match) {
                rc = FOUND;
                rh = (int64_t)(bucket * (uint64_t)(BW / V) + (__ffs(match) - 1));
            } else {
                uint32_t empty = ~occ & ALL;
                uint32_t* base = T.data + bucket * (uint64_t)BW;
                while (empty) {
                    int s = __ffs(empty) - 1;
                    uint32_t old[V];
                    if (SlotCas<V>::cas(base + s * V, km, old)) {
                        rc = INSERTED;
                        rh = (int64_t)(bucket * (uint64_t)(BW / V) + s);
                        if (T.track_status) T.status[bucket * (uint64_t)T.stride + s] = NEW;
                        break;
                    }
                    bool eq = true;
#pragma unroll
                    for (int w = 0; w < V; w++) eq = eq && (old[w] == km[w]);
                    if (eq) {
                        rc = FOUND;
                        rh = (int64_t)(bucket * (uint64_t)(BW / V) + s);
                        break;
                    }
                    empty &= ~(1u << s);
                }
            }
        }
        // broadcast the leader's verdict to its group
        rc = __shfl_sync(FULLMASK, rc, leader);
        rh = (int64_t)__shfl_sync(FULLMASK, (unsigned long long)rh, leader);
        if (todo && rc >= 0) {
            code = rc;
            hd = rh;
        }
    }
    if (active && code < 0) code = TABLE_FULL;
    *handle = active ? hd : -1;
    return code;
}

// Claim in a bucket whose masks the group has already computed: runs in
// the group leader only.  rc = -1 when the bucket is full.
template <int BW, int V>
__device__ __forceinline__ void leader_resolve(const TableDesc& T, uint64_t bucket, uint32_t occ,
                                               uint32_t match, const uint32_t* km, int* rc,
                                               int64_t* rh) {
    constexpr int SPB = BW / V;
    constexpr uint32_t ALL = SPB >= 32 ? 0xffffffffu : ((1u << SPB) - 1u);
    if (match) {
        *rc = FOUND;
        *rh = (int64_t)(bucket * (uint64_t)SPB + (__ffs(match) - 1));
        return;
    }
    uint32_t empty = ~occ & ALL;
    uint32_t* base = T.data + bucket * (uint64_t)BW;
    while (empty) {
        const int s = __ffs(empty) - 1;
        uint32_t old[V];
        if (SlotCas<V>::cas(base + s * V, km, old)) {
            *rc = INSERTED;
            *rh = (int64_t)(bucket * (uint64_t)SPB + s);
            return;
        }
        bool eq = true;
#pragma unroll
        for (int w = 0; w < V; w++) eq = eq && (old[w] == km[w]);
        if (eq) {
            *rc = FOUND;
            *rh = (int64_t)(bucket * (uint64_t)SPB + s);
            return;
        }
        empty &= ~(1u << s);
    }
    *rc = -1;
}

// ----------------------------------------------------- batched probing
//
// A warp probes KB = 32*M keys per batch.  Lane l owns keys l + 32*m
// (m < M): it computes their fold and first bucket once.  Lane group grp
// (G lanes) then handles keys e = u*R + grp for u < U = M*G (R = 32/G
// groups), pulling each key's words and bucket from its owner lane
// ((u % G)*R + grp, slot u / G -- both compile-time in u) by shuffle, and
// issues all U*CPL 16-byte bucket loads before consuming any.  The group
// leader resolves each key (FOUND / CAS-insert / bucket full); keys whose
// first bucket is full continue through hash functions 1..K-1 with
// probe_mark (rare below the load cliff).
template <int BW, int G>
struct ProbeShape {
    static constexpr int CH = BW / 4;     // 16-byte chunks per bucket
    static constexpr int CPL = CH / G;    // chunks per lane per key
    static constexpr int M = BW >= 32 ? 1 : (4 / CH > 1 ? 4 / CH : 1);  // owned keys per lane
    static constexpr int U = M * G;       // keys per lane group per batch
    static constexpr int R = 32 / G;      // lane groups per warp
    static constexpr int KB = 32 * M;     // keys per warp per batch
};

template <int BW, int V, int G>
__device__ __forceinline__ void probe_batch(const TableDesc& T,
                                            const uint32_t (&own_key)[ProbeShape<BW, G>::M][V],
                                            const bool (&own_act)[ProbeShape<BW, G>::M],
                                            uint32_t (&key)[ProbeShape<BW, G>::U][V],
                                            bool (&act)[ProbeShape<BW, G>::U],
                                            int (&code)[ProbeShape<BW, G>::U],
                                            int64_t (&hd)[ProbeShape<BW, G>::U]) {
    using S = ProbeShape<BW, G>;
    constexpr int M = S::M, U = S::U, R = S::R, CPL = S::CPL;
    constexpr int SPC = 4 / V;
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);
    const int grp = lane / G;
    const int leader = lane & ~(G - 1);
    uint64_t own_b[M];
#pragma unroll
    for (int m = 0; m < M; m++) own_b[m] = own_act[m] ? bucket_of(T, fold<V>(T.salt, own_key[m]), 0) : 0;
    uint4 ch[U][CPL];
    uint64_t bucket[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
        const int src = (u % G) * R + grp;
        const int m = u / G;
        act[u] = __shfl_sync(FULLMASK, own_act[m] ? 1 : 0, src) != 0;
        bucket[u] = __shfl_sync(FULLMASK, (unsigned long long)own_b[m], src);
#pragma unroll
        for (int w = 0; w < V; w++) key[u][w] = __shfl_sync(FULLMASK, own_key[m][w], src);
        if (act[u]) {
            const uint32_t* base = T.data + bucket[u] * (uint64_t)BW;
#pragma unroll
            for (int j = 0; j < CPL; j++) ch[u][j] = ldcg4(base + 4 * (gl + j * G));
        }
    }
    // masks of every key first, then the leaders' first-choice CASes issued
    // back to back (independent atomics overlap instead of paying one L2
    // round trip per key), then the verdicts; a lost first CAS re-judges
    // the remaining EMPTY slots serially (rare).
    constexpr int SPB = BW / V;
    constexpr uint32_t ALL = SPB >= 32 ? 0xffffffffu : ((1u << SPB) - 1u);
    uint32_t occ[U], match[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
        uint32_t km[V];
#pragma unroll
        for (int w = 0; w < V; w++) km[w] = key[u][w] | (w == (int)T.mark_word ? T.mark : 0u);
        occ[u] = 0;
        match[u] = 0;
        if (act[u]) {
#pragma unroll
            for (int j = 0; j < CPL; j++) {
                const uint32_t w4[4] = {ch[u][j].x, ch[u][j].y, ch[u][j].z, ch[u][j].w};
                const int c = gl + j * G;
#pragma unroll
                for (int t = 0; t < SPC; t++) {
                    const int sl = c * SPC + t;
                    uint32_t ob = 0;
                    bool mm = true;
#pragma unroll
                    for (int w = 0; w < V; w++) {
                        ob |= w4[t * V + w] & (w == (int)T.mark_word ? T.mark : 0u);
                        mm = mm && (w4[t * V + w] == km[w]);
                    }
                    occ[u] |= (ob != 0u ? 1u : 0u) << sl;
                    match[u] |= (mm ? 1u : 0u) << sl;
                }
            }
        }
#pragma unroll
        for (int o = 1; o < G; o <<= 1) {
            occ[u] |= __shfl_xor_sync(FULLMASK, occ[u], o);
            match[u] |= __shfl_xor_sync(FULLMASK, match[u], o);
        }
    }
    int rc[U], slot[U];
    uint32_t old[U][V];
#pragma unroll
    for (int u = 0; u < U; u++) {
        rc[u] = -1;
        slot[u] = -1;
        if (act[u] && gl == 0) {
            if (match[u]) {
                rc[u] = FOUND;
                slot[u] = __ffs(match[u]) - 1;
            } else {
                const uint32_t empty = ~occ[u] & ALL;
                if (empty) {
                    uint32_t km[V];
#pragma unroll
                    for (int w = 0; w < V; w++) km[w] = key[u][w] | (w == (int)T.mark_word ? T.mark : 0u);
                    slot[u] = __ffs(empty) - 1;
                    SlotCas<V>::cas(T.data + bucket[u] * (uint64_t)BW + slot[u] * V, km, old[u]);
                    rc[u] = -3;  // CAS in flight
                }
            }
        }
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
        int64_t rh = -1;
        if (rc[u] == -3) {
            uint32_t km[V];
            bool zero = true, eq = true;
#pragma unroll
            for (int w = 0; w < V; w++) {
                km[w] = key[u][w] | (w == (int)T.mark_word ? T.mark : 0u);
                zero = zero && old[u][w] == 0u;
                eq = eq && old[u][w] == km[w];
            }
            if (zero) {
                rc[u] = INSERTED;
            } else if (eq) {
                rc[u] = FOUND;
            } else {
                // lost the first EMPTY slot to another key: the rest in order
                const uint32_t rest = ~occ[u] & ALL & ~((2u << slot[u]) - 1u);
                leader_resolve<BW, V>(T, bucket[u], ~rest & ALL, 0u, km, &rc[u], &rh);
                slot[u] = -1;
            }
        }
        if (slot[u] >= 0) rh = (int64_t)(bucket[u] * (uint64_t)SPB + slot[u]);
        int r = rc[u];
        if (G > 1) r = __shfl_sync(FULLMASK, r, leader);
        code[u] = act[u] ? r : -1;
        hd[u] = rh;
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
        const bool need = act[u] && code[u] < 0;
        if (__any_sync(FULLMASK, need)) {
            int64_t x;
            const int c = probe_mark<BW, V, G>(T, need, key[u], fold<V>(T.salt, key[u]), &x, 1);
            if (need) {
                code[u] = c;
                hd[u] = x;
            }
        }
    }
}

// ---------------------------------------------- MODE_STATUS per-lane probe
__device__ __forceinline__ uint32_t status_word_cas_byte(uint8_t* cell, uint32_t from, uint32_t to,
                                                         uint32_t* seen) {
    // CAS one status byte from `from` to `to` via its aligned 32-bit word.
    uintptr_t addr = reinterpret_cast<uintptr_t>(cell);
    uint32_t* w = reinterpret_cast<uint32_t*>(addr & ~uintptr_t(3));
    const int sh = (int)(addr & 3) * 8;
    uint32_t cur = __ldcg(w);
    for (;;) {
        uint32_t b = (cur >> sh) & 0xffu;
        if (b != from) {
            *seen = b;
            return 0;
        }
        uint32_t nv = (cur & ~(0xffu << sh)) | (to << sh);
        uint32_t prev = atomicCAS(w, cur, nv);
        if (prev == cur) {
            *seen = from;
            return 1;
        }
        cur = prev;
    }
}

__device__ __forceinline__ uint32_t ld_status_acquire(const uint8_t* cell) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u8 %0, [%1];" : "=r"(v) : "l"(cell) : "memory");
    return v & 0xffu;
}

__device__ __forceinline__ void st_status_release(uint8_t* cell, uint32_t v) {
    asm volatile("st.release.gpu.global.u8 [%0], %1;" ::"l"(cell), "r"(v) : "memory");
}

// find_or_insert, hashtable.py:224-280, one lane per key, any vlen.
__device__ __forceinline__ int probe_status(const TableDesc& T, const uint32_t* key, uint64_t h,
                                            int64_t* handle) {
    const int V = (int)T.vlen;
    for (int i = 0; i < (int)T.k; i++) {
        uint64_t bucket = bucket_of(T, h, i);
        uint8_t* sb = T.status + bucket * (uint64_t)T.stride;
        uint32_t* db = T.data + bucket * (uint64_t)T.bw;
        for (int j = 0; j < (int)T.spb; j++) {
            uint32_t st = ld_status_acquire(sb + j);
            if (st == EMPTY) {
                uint32_t seen;
                if (status_word_cas_byte(sb + j, EMPTY, CLAIMED, &seen)) {
                    uint32_t* d = db + T.offsets[j];
                    for (int w = 0; w < V; w++) __stcg(d + w, key[w]);
                    __threadfence();
                    st_status_release(sb + j, NEW);
                    *handle = (int64_t)(bucket * (uint64_t)T.spb + j);
                    return INSERTED;
                }
                st = seen;
            }
            while (st == CLAIMED) {  // _wait_published, hashtable.py:282-294
                __nanosleep(64);
                st = ld_status_acquire(sb + j);
            }
            const uint32_t* d = db + T.offsets[j];
            bool eq = true;
            for (int w = 0; w < V && eq; w++) eq = __ldcg(d + w) == key[w];
            if (eq) {
                *handle = (int64_t)(bucket * (uint64_t)T.spb + j);
                return FOUND;
            }
        }
    }
    *handle = -1;
    return TABLE_FULL;
}

// Is slot (bucket, j) occupied (published)?
__device__ __forceinline__ bool slot_occupied(const TableDesc& T, uint64_t bucket, int j) {
    if (T.mode == MODE_STATUS) return T.status[bucket * (uint64_t)T.stride + j] >= NEW;
    const uint32_t* d = T.data + bucket * (uint64_t)T.bw + T.offsets[j];
    return (__ldcg(d + T.mark_word) & T.mark) != 0u;
}

}  // namespace gx
