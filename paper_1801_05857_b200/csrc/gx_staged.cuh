// gx_staged.cuh -- FINDORPUT with the bucket loads staged in shared memory.
//
// The register-group probe (probe_batch, gx_device.cuh) holds every loaded
// bucket in registers, so a warp can keep only ~32 buckets in flight and
// the level kernel is latency bound (profiles/README.md, r1b: 19% of DRAM
// peak, long-scoreboard stalls).  Here a warp stages a whole batch of KB
// first buckets into its shared-memory slice with cp.async (LDGSTS,
// L2-cached, no registers held while in flight), waits once, and then
// every lane resolves its own keys from shared memory:
//
//   1. lane l owns keys l, l+32, ... of the batch: fold, first bucket
//      (hashtable.py:205-217), bucket index -> per-warp smem array
//   2. the warp copies the KB buckets (BW/4 16-byte chunks each, chunk j
//      of key k at position j ^ (k mod CH): conflict-free LDS.128 later)
//   3. each lane walks its buckets' slots in order: first slot equal to
//      the key -> FOUND; first EMPTY slot -> CAS candidate (occupied slots
//      are a bucket prefix, hashtable.py:229-231); none -> bucket full
//   4. all candidates' CASes are issued back to back, then judged: lost to
//      the same key -> FOUND, lost to another -> walk the rest of the
//      bucket from global memory (rare)
//   5. keys whose bucket was full repeat 2-4 with the next hash function,
//      again all staged at once (hashtable.py:237-280); after K full
//      buckets -> TABLE_FULL
//
// Slot j of a bucket sits at word j*V for every layout the in-band mode
// allows (vlen 1/2/4: the half layout's second half starts at bw/2, which
// is exactly spb/2 slots in), so a bucket is scanned as a contiguous array.
#pragma once
#include "gx_device.cuh"

#ifndef GX_STAGE_BYTES
#define GX_STAGE_BYTES 8192  // shared-memory bucket staging per warp
#endif
#ifndef GX_STAGE_KB_MAX
#define GX_STAGE_KB_MAX 32  // keys per staged batch at most (B200 sweeps: 3 blocks x 32 > 2 blocks x 64)
#endif
#ifndef GX_TMA
#define GX_TMA 0  // 1: stage buckets with one bulk copy (TMA) per key instead of BW/4 cp.async (B200: 5-10% slower, profiles/README.md)
#endif

namespace gx {

__device__ __forceinline__ uint32_t lanemask_lt_() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// A slot's words as one single-copy-atomic read (a torn read of a slot that
// is being claimed could look like "another key" and let the key be
// inserted twice further on).  V = 4 reads through a no-op CAS.
template <int V>
__device__ __forceinline__ void load_slot(uint32_t* p, uint32_t* out) {
    if (V == 1) {
        out[0] = __ldcg(p);
    } else if (V == 2) {
        const unsigned long long x = __ldcg(reinterpret_cast<const unsigned long long*>(p));
        out[0] = (uint32_t)x;
        out[1] = (uint32_t)(x >> 32);
    } else {
        const uint32_t zero[V] = {};
        SlotCas<V>::cas(p, zero, out);
    }
}

// One key, one lane: continue FINDORPUT in `bucket` from slot s0 on, reading
// slots from global memory (after a lost CAS).  rc = -1 if the bucket fills.
template <int BW, int V>
__device__ __forceinline__ int resolve_lane_from(const TableDesc& T, uint64_t bucket, int s0,
                                                 const uint32_t* km, int64_t* handle) {
    constexpr int SPB = BW / V;
    uint32_t* base = T.data + bucket * (uint64_t)BW;
    for (int s = s0; s < SPB; s++) {
        uint32_t cur[V];
        load_slot<V>(base + s * V, cur);
        bool zero = true;
#pragma unroll
        for (int w = 0; w < V; w++) zero = zero && cur[w] == 0u;
        if (zero) {
            if (SlotCas<V>::cas(base + s * V, km, cur)) {
                *handle = (int64_t)(bucket * (uint64_t)SPB + s);
                return INSERTED;
            }
        }
        bool eq = true;
#pragma unroll
        for (int w = 0; w < V; w++) eq = eq && cur[w] == km[w];
        if (eq) {
            *handle = (int64_t)(bucket * (uint64_t)SPB + s);
            return FOUND;
        }
    }
    return -1;
}

// Hash functions i0..K-1 for one key, one lane (hashtable.py:237-280).
template <int BW, int V>
__device__ __forceinline__ int probe_lane(const TableDesc& T, const uint32_t* km, uint64_t h, int i0,
                                          int64_t* handle) {
    for (int i = i0; i < (int)T.k; i++) {
        const int rc = resolve_lane_from<BW, V>(T, bucket_of(T, h, i), 0, km, handle);
        if (rc >= 0) return rc;
    }
    *handle = -1;
    return TABLE_FULL;
}

// KBX > 0 overrides the batch size (a 128-key absorb batch was tried on the
// B200: 18% slower than 3 blocks x 8 warps x 32 keys, see profiles/README.md)
template <int BW, int V, int KBX = 0>
struct Staged {
    static constexpr int CH = BW / 4;                 // 16-byte chunks per bucket
    static constexpr int SPB = BW / V;                // slots per bucket
    static constexpr int SPC = 4 / V;                 // slots per chunk
    static constexpr int KB = KBX > 0 ? KBX
                              : (GX_STAGE_BYTES / (4 * BW) > GX_STAGE_KB_MAX ? GX_STAGE_KB_MAX
                                                                             : GX_STAGE_BYTES / (4 * BW));
    static constexpr int STAGE_BYTES = KB * 4 * BW;   // per warp
    static constexpr int KPL = KB / 32;               // keys per lane per batch
    // u64 words per warp of the index array: KB bucket indices, then the
    // warp's TMA mbarrier and its phase
    static constexpr int SB_STRIDE = KB + 2;
};

// ---------------------------------------------------- TMA bucket staging
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// once per warp before its first probe_staged: the warp's mbarrier (one
// arrival per round: lane 0's expect_tx) and its phase bit
__device__ __forceinline__ void staged_init(unsigned long long* sbkt, int kb) {
#if GX_TMA
    if ((threadIdx.x & 31) == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(sbkt + kb)) : "memory");
        sbkt[kb + 1] = 0ull;
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
#endif
}

__device__ __forceinline__ void tma_expect(unsigned long long* mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mbar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void tma_load(void* dst, const void* src, uint32_t bytes, unsigned long long* mbar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(mbar))
        : "memory");
}

__device__ __forceinline__ void tma_wait(unsigned long long* mbar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(mbar)),
        "r"(parity)
        : "memory");
}

#ifndef GX_REFILL
#define GX_REFILL 1  // one key per lane, lanes refilled as their keys resolve (see probe_refill)
#endif
#ifndef GX_DEFER_CAS
// 1: probe_refill judges a claim CAS one round after issuing it (the warp
// does not wait for the atomic; the lane sits out one round).  Exact (the
// GPU suite passes with it on), but slower on B200: ring19 1.85 vs 1.92,
// ring16 2.93 vs 3.07 ·10^9 states/s, peterson6 level 156 vs 152 ms
// (profiles/round2/s2zu_*): a lane idle for a whole round costs more than
// the CAS round trip the warp would otherwise wait for.
#define GX_DEFER_CAS 0
#endif
#ifndef GX_PREFETCH
// 1: probe_refill prefetches the next round's first buckets into L2 while
// a round's loads fly.  Exact, but slower on B200: ring19 1.63 vs 1.92,
// ring16 2.57 vs 3.07 ·10^9 states/s (peterson6 level 150 vs 152 ms),
// profiles/round2/s2zr_*: the extra fold + bucket per key and round and the
// second request per probe cost more than the latency they hide.
#define GX_PREFETCH 0
#endif

// a 128-byte line into L2: a 16-byte cp.async with the 128 B L2 prefetch
// size into a dump slot (a per-lane instruction; the bulk L2 prefetch
// takes a uniform address and compiles to a 32-pass loop per warp)
__device__ __forceinline__ void prefetch_l2_128(void* dump, const void* gmem) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(dump);
    asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// FINDORPUT of keys q[0, m) with every lane owning one key at a time and a
// round = one bucket per lane: all 32 buckets of a round are staged with
// cp.async at once, each lane resolves its key from shared memory, and a
// lane whose key is done (FOUND, INSERTED, TABLE_FULL) takes the next key
// of q while the lanes whose bucket was full go on to their next hash
// function in the same round.  The batch-synchronous version
// (probe_staged below with GX_REFILL 0) ran a whole extra memory round
// for the few keys of a batch of 32 that needed a second bucket -- at load
// 0.75, 95% of batches; here those keys share a round with fresh keys.
// Same results: each key's probe sequence and CAS protocol are unchanged
// (hashtable.py:224-280).  INSERTED keys are written, compacted, to the
// front of q (always below the next key to read); returns their number.
template <int BW, int V>
__device__ __forceinline__ uint32_t probe_refill(const TableDesc& T, uint32_t* q, uint32_t m, uint4* stage,
                                                 unsigned long long* sbkt, uint32_t* full,
                                                 uint32_t* nprobe = nullptr) {
    constexpr int CH = BW / 4, SPC = 4 / V;
    constexpr unsigned long long SKIP = ~0ull;
    const int lane = threadIdx.x & 31;
    const uint32_t mark_lo = T.mark;
    uint32_t n_ins = 0;
    // lane state: its key (with the mark), fold, hash function index
    uint32_t km[V];
    uint64_t h = 0;
    int r = 0;
    bool has = (uint32_t)lane < m;
    uint32_t nxt = min(m, 32u);  // next key of q to hand out
    {
        uint32_t key[V];
#pragma unroll
        for (int w = 0; w < V; w++) key[w] = has ? q[lane * V + w] : 0u;
        h = fold<V>(T.salt, key);
#pragma unroll
        for (int w = 0; w < V; w++) km[w] = key[w] | (w == (int)T.mark_word ? mark_lo : 0u);
    }
#if GX_DEFER_CAS
    bool pend = false;  // this lane's claim CAS is in flight (issued last round)
    uint32_t pold[V];
    int pslot = 0;
#pragma unroll
    for (int w = 0; w < V; w++) pold[w] = 0u;
#endif
    while (__any_sync(FULLMASK, has)) {
#if GX_DEFER_CAS
        const bool ld = has && !pend;  // lanes that stage a bucket this round
#else
        const bool ld = has;
#endif
        const uint64_t bkt = has ? bucket_of(T, h, r) : 0;
        sbkt[lane] = ld ? bkt : SKIP;
        if (nprobe) *nprobe += ld ? 1u : 0u;
        __syncwarp();
#pragma unroll
        for (int it = 0; it < CH; it++) {
            const uint32_t c = it * 32 + lane;
            const uint32_t k = c / CH, j = c % CH;
            const unsigned long long b = sbkt[k];
            if (b != SKIP) cp_async16(stage + k * CH + (j ^ (k & (CH - 1))), T.data + b * (uint64_t)BW + 4 * j);
        }
#if GX_PREFETCH
        // while the round's loads fly: the first buckets of the next 32
        // queued keys (the keys lanes take when theirs resolve) into L2, so
        // the round that stages them finds them there; their folds travel
        // to the taking lanes by shuffle.  The prefetches are their own
        // cp.async group, which the round does not wait for.
        __shared__ uint4 pf_dump[32];  // never read
        cp_async_commit();
        uint64_t hn = 0;
        if (nxt + lane < m) {
            uint32_t key[V];
#pragma unroll
            for (int w = 0; w < V; w++) key[w] = q[(nxt + lane) * V + w];
            hn = fold<V>(T.salt, key);
            prefetch_l2_128(pf_dump + lane, T.data + bucket_of(T, hn, 0) * (uint64_t)BW);
        }
        cp_async_commit();
        cp_async_wait1();
#else
        cp_async_wait_all();
#endif
        __syncwarp();
        int rc = -1, slot = -1;
        if (ld) {
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
                        rc = -3;  // CAS candidate
                        slot = j * SPC + t;
                    }
                }
            }
        }
        __syncwarp();  // stage and sbkt are free again
#if GX_DEFER_CAS
        // the claim CAS is judged one round after it was issued: the warp
        // does not wait for the atomic's round trip, the lane just sits out
        // one round's load.  Same judgement as below.
        if (pend) {
            bool zero = true, eq = true;
#pragma unroll
            for (int w = 0; w < V; w++) {
                zero = zero && pold[w] == 0u;
                eq = eq && pold[w] == km[w];
            }
            if (zero) {
                rc = INSERTED;
            } else if (eq) {
                rc = FOUND;
            } else {  // lost the slot to another key: the rest of the bucket
                int64_t hd;
                rc = resolve_lane_from<BW, V>(T, bkt, pslot + 1, km, &hd);
            }
            pend = false;
        }
        if (rc == -3) {
            SlotCas<V>::cas(T.data + bkt * (uint64_t)BW + slot * V, km, pold);
            pslot = slot;
            pend = true;
            rc = -2;  // in flight: neither done nor a full bucket
        }
#else
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
            } else {  // lost the slot to another key: the rest of the bucket
                int64_t hd;
                rc = resolve_lane_from<BW, V>(T, bkt, slot + 1, km, &hd);
            }
        }
#endif
        bool done = false;
        if (has) {
            if (rc == -1 && ++r >= (int)T.k) rc = TABLE_FULL;  // all K buckets full
            done = rc >= 0;
        }
        *full += (done && rc == TABLE_FULL) ? 1u : 0u;
        // INSERTED keys to the front of q (positions below nxt: consumed)
        const bool ins = done && rc == INSERTED;
        const uint32_t im = __ballot_sync(FULLMASK, ins);
        if (ins) {
            const uint32_t p = n_ins + __popc(im & lanemask_lt_());
#pragma unroll
            for (int w = 0; w < V; w++) q[p * V + w] = km[w] & ~(w == (int)T.mark_word ? mark_lo : 0u);
        }
        n_ins += __popc(im);
        // refill the lanes that finished with the next keys of q
        const uint32_t dm = __ballot_sync(FULLMASK, done);
#if GX_PREFETCH
        const uint64_t hs = __shfl_sync(FULLMASK, hn, (int)(__popc(dm & lanemask_lt_()) & 31));
#endif
        if (done) {
            const uint32_t idx = nxt + __popc(dm & lanemask_lt_());
            has = idx < m;
            if (has) {
                uint32_t key[V];
#pragma unroll
                for (int w = 0; w < V; w++) key[w] = q[idx * V + w];
#if GX_PREFETCH
                h = hs;
#else
                h = fold<V>(T.salt, key);
#endif
#pragma unroll
                for (int w = 0; w < V; w++) km[w] = key[w] | (w == (int)T.mark_word ? mark_lo : 0u);
                r = 0;
            }
        }
        nxt = min(m, nxt + __popc(dm));
        __syncwarp();
    }
#if GX_PREFETCH
    cp_async_wait0();  // the last prefetch group
#endif
    return n_ins;
}

// FINDORPUT of keys q[0, m) (V words each, shared memory), KB at a time.
// INSERTED keys are written back, compacted, to the front of q (a key is
// only ever written at or below the position it was read from); returns
// their number.  *full counts (per lane) the keys that hit TABLE_FULL.  stage: this
// warp's STAGE_BYTES of shared memory; sbkt: its KB bucket indices.
template <int BW, int V, int KBX = 0>
__device__ __forceinline__ uint32_t probe_staged(const TableDesc& T, uint32_t* q, uint32_t m,
                                                 uint4* stage, unsigned long long* sbkt,
                                                 uint32_t* full, uint32_t* nprobe = nullptr) {
    using S = Staged<BW, V, KBX>;
    constexpr int KB = S::KB, KPL = S::KPL, CH = S::CH, SPC = S::SPC;
    constexpr unsigned long long SKIP = ~0ull;
#if GX_REFILL && !GX_TMA
    if constexpr (KPL == 1) return probe_refill<BW, V>(T, q, m, stage, sbkt, full, nprobe);
#endif
    const int lane = threadIdx.x & 31;
    uint32_t n_ins = 0;
    for (uint32_t r0 = 0; r0 < m; r0 += KB) {
        const uint32_t nb = min((uint32_t)KB, m - r0);
        uint32_t km[KPL][V];
        uint64_t h[KPL], bkt[KPL];
        bool act[KPL], pend[KPL];
        int rc[KPL];
#pragma unroll
        for (int i = 0; i < KPL; i++) {
            const uint32_t k = lane + 32 * i;
            act[i] = k < nb;
            pend[i] = act[i];
            rc[i] = -1;
            uint32_t key[V];
#pragma unroll
            for (int w = 0; w < V; w++) key[w] = act[i] ? q[(r0 + k) * V + w] : 0u;
            h[i] = fold<V>(T.salt, key);
#pragma unroll
            for (int w = 0; w < V; w++) km[i][w] = key[w] | (w == (int)T.mark_word ? T.mark : 0u);
        }
        // hash function hi for every key still unresolved (hi = 0: all of
        // them; later rounds only the keys whose bucket was full), each
        // round with all of its bucket loads in flight at once
        for (int hi = 0; hi < (int)T.k; hi++) {
            bool any = false;
#pragma unroll
            for (int i = 0; i < KPL; i++) {
                const uint32_t k = lane + 32 * i;
                bkt[i] = pend[i] ? bucket_of(T, h[i], hi) : 0;
                sbkt[k] = pend[i] ? bkt[i] : SKIP;
                any |= pend[i];
                if (nprobe) *nprobe += pend[i] ? 1u : 0u;  // bucket loads (the bench's probes/op)
            }
            if (!__any_sync(FULLMASK, any)) break;
            __syncwarp();
            int slot[KPL];
            uint32_t old[KPL][V];
#if GX_TMA
            // one bulk copy per pending key, completing on the warp's
            // mbarrier (its expected bytes set first by lane 0)
            {
                unsigned long long* mbar = sbkt + KB;
                uint32_t np = 0;
#pragma unroll
                for (int i = 0; i < KPL; i++) np += __popc(__ballot_sync(FULLMASK, pend[i]));
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // prior generic stage use first
                __syncwarp();
                if (lane == 0) tma_expect(mbar, np * (uint32_t)(16 * CH));
                __syncwarp();
#pragma unroll
                for (int i = 0; i < KPL; i++)
                    if (pend[i]) tma_load(stage + (lane + 32 * i) * CH, T.data + bkt[i] * (uint64_t)BW, 16 * CH, mbar);
                const uint32_t ph = (uint32_t)sbkt[KB + 1];
                tma_wait(mbar, ph);
                __syncwarp();
                if (lane == 0) sbkt[KB + 1] = ph ^ 1u;
            }
            // walk every pending bucket from shared memory: all chunks, each
            // lane starting at a rotated chunk (conflict-free 16-byte reads
            // of unswizzled buckets); a match anywhere -> FOUND, else the
            // lowest EMPTY slot is the CAS candidate (occupied slots are a
            // prefix, hashtable.py:229-231; a stale view only costs a lost CAS)
#pragma unroll
            for (int i = 0; i < KPL; i++) {
                const uint32_t k = lane + 32 * i;
                slot[i] = -1;
                if (!pend[i]) continue;
                int found = -1, empty = 1 << 20;
                const int rot = (int)((k * CH) / 8);
#pragma unroll
                for (int j = 0; j < CH; j++) {
                    const int jj = (j + rot) & (CH - 1);
                    const uint4 c4 = stage[k * CH + jj];
                    const uint32_t w4[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
                    for (int t = 0; t < SPC; t++) {
                        bool zero = true, eq = true;
#pragma unroll
                        for (int w = 0; w < V; w++) {
                            zero = zero && w4[t * V + w] == 0u;
                            eq = eq && w4[t * V + w] == km[i][w];
                        }
                        const int sl = jj * SPC + t;
                        if (eq) found = sl;
                        if (zero && sl < empty) empty = sl;
                    }
                }
                if (found >= 0) {
                    rc[i] = FOUND;
                    slot[i] = found;
                } else if (empty < S::SPB) {
                    rc[i] = -3;  // CAS candidate
                    slot[i] = empty;
                }
            }
#else
            // stage the buckets: chunk c = key c / CH, part c % CH
#pragma unroll
            for (int it = 0; it < KPL * CH; it++) {
                const uint32_t c = it * 32 + lane;
                const uint32_t k = c / CH, j = c % CH;
                const unsigned long long b = sbkt[k];
                if (b != SKIP)
                    cp_async16(stage + k * CH + (j ^ (k & (CH - 1))), T.data + b * (uint64_t)BW + 4 * j);
            }

            cp_async_wait_all();
            __syncwarp();
            // walk each pending bucket from shared memory
#pragma unroll
            for (int i = 0; i < KPL; i++) {
                const uint32_t k = lane + 32 * i;
                slot[i] = -1;
                if (!pend[i]) continue;
                for (int j = 0; j < CH && rc[i] == -1; j++) {
                    const uint4 c4 = stage[k * CH + (j ^ (k & (CH - 1)))];
                    const uint32_t w4[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
                    for (int t = 0; t < SPC; t++) {
                        if (rc[i] != -1) break;
                        bool zero = true, eq = true;
#pragma unroll
                        for (int w = 0; w < V; w++) {
                            zero = zero && w4[t * V + w] == 0u;
                            eq = eq && w4[t * V + w] == km[i][w];
                        }
                        if (eq) {
                            rc[i] = FOUND;
                            slot[i] = j * SPC + t;
                        } else if (zero) {
                            rc[i] = -3;  // CAS candidate
                            slot[i] = j * SPC + t;
                        }
                    }
                }
            }
#endif
            __syncwarp();  // stage and sbkt are free again
            // the candidates' CASes back to back
#pragma unroll
            for (int i = 0; i < KPL; i++)
                if (pend[i] && rc[i] == -3)
                    SlotCas<V>::cas(T.data + bkt[i] * (uint64_t)BW + slot[i] * V, km[i], old[i]);
#pragma unroll
            for (int i = 0; i < KPL; i++) {
                if (!pend[i]) continue;
                if (rc[i] == -3) {
                    int64_t hd;
                    bool zero = true, eq = true;
#pragma unroll
                    for (int w = 0; w < V; w++) {
                        zero = zero && old[i][w] == 0u;
                        eq = eq && old[i][w] == km[i][w];
                    }
                    if (zero)
                        rc[i] = INSERTED;
                    else if (eq)
                        rc[i] = FOUND;
                    else  // lost the slot to another key: the rest of the bucket
                        rc[i] = resolve_lane_from<BW, V>(T, bkt[i], slot[i] + 1, km[i], &hd);
                }
                pend[i] = rc[i] == -1;  // bucket full: next hash function
            }
        }
        bool ins[KPL];
#pragma unroll
        for (int i = 0; i < KPL; i++) {
            if (act[i] && rc[i] == -1) rc[i] = TABLE_FULL;  // all K buckets full
            ins[i] = act[i] && rc[i] == INSERTED;
            *full += (act[i] && rc[i] == TABLE_FULL) ? 1u : 0u;
        }
        // INSERTED keys to the front of q, in key order
#pragma unroll
        for (int i = 0; i < KPL; i++) {
            const uint32_t msk = __ballot_sync(FULLMASK, ins[i]);
            if (ins[i]) {
                const uint32_t p = n_ins + __popc(msk & lanemask_lt_());
#pragma unroll
                for (int w = 0; w < V; w++) q[p * V + w] = km[i][w] & ~(w == (int)T.mark_word ? T.mark : 0u);
            }
            n_ins += __popc(msk);
        }
        __syncwarp();
    }
    return n_ins;
}

}  // namespace gx
