// gx_expand.cuh -- successor generation on packed state vectors
// (network.py:184-238 semantics, restated on the device CSR).
#pragma once
#include "gx_internal.h"

namespace gx {

// s[w] with a runtime w, as a select chain so the state stays in registers
template <int V>
__device__ __forceinline__ uint32_t word_at(const uint32_t* s, uint32_t w) {
    uint32_t r = s[0];
#pragma unroll
    for (int i = 1; i < V; i++) r = (w == (uint32_t)i) ? s[i] : r;
    return r;
}

template <int V>
__device__ __forceinline__ uint32_t field_get(const uint32_t* s, uint32_t word, uint32_t shift,
                                              uint32_t mask) {
    return (word_at<V>(s, word) >> shift) & mask;
}

// Does rule r' produce target t from source s?  True iff t differs from s
// only in r's participants and each participant's value in t is one of its
// rule destinations at its value in s (network.py:213-237).
template <int V>
__device__ __forceinline__ bool rule_generates(const NetDesc& N, uint32_t r, const uint32_t* s,
                                               const uint32_t* t) {
    if (V <= 4 && N.rmask) {
        // t may differ from s only in r's participants
        const uint4 m = __ldg(&N.rmask[r]);
        const uint32_t allowed[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
        for (int w = 0; w < (V < 4 ? V : 4); w++)
            if ((s[w] ^ t[w]) & ~allowed[w]) return false;
    }
    const uint4 rl = __ldg(&N.rules[r]);
    if (V > 4 || !N.rmask) {
        uint32_t allowed[V];
#pragma unroll
        for (int w = 0; w < V; w++) allowed[w] = 0;
        for (uint32_t k = 0; k < rl.x; k++) {
            const uint4 pt = __ldg(&N.parts[rl.y + k]);
#pragma unroll
            for (int w = 0; w < V; w++)
                if ((uint32_t)w == pt.y) allowed[w] |= pt.w << pt.z;
        }
#pragma unroll
        for (int w = 0; w < V; w++)
            if ((s[w] ^ t[w]) & ~allowed[w]) return false;
    }
    for (uint32_t k = 0; k < rl.x; k++) {
        const uint4 pt = __ldg(&N.parts[rl.y + k]);
        const uint32_t sq = field_get<V>(s, pt.y, pt.z, pt.w);
        const uint32_t tq = field_get<V>(t, pt.y, pt.z, pt.w);
        const uint2 l = __ldg(&N.rq[pt.x + sq]);
        bool in = false;
        for (uint32_t d = 0; d < l.y && !in; d++) in = __ldg(&N.rdst[l.x + d]) == tq;
        if (!in) return false;
    }
    return true;
}

// Build the target of combination `c` of rule `rl` from s into t.
template <int V>
__device__ __forceinline__ void rule_target(const NetDesc& N, const uint4 rl, uint32_t c,
                                            const uint32_t* s, uint32_t* t) {
#pragma unroll
    for (int w = 0; w < V; w++) t[w] = s[w];
    if (c == 0) {
        // combination 0 (the only one when every participant has a single
        // destination, the common case): every digit is 0, no division
        for (uint32_t k = 0; k < rl.x; k++) {
            const uint4 pt = __ldg(&N.parts[rl.y + k]);
            const uint2 l = __ldg(&N.rq[pt.x + field_get<V>(s, pt.y, pt.z, pt.w)]);
            const uint32_t dst = __ldg(&N.rdst[l.x]);
#pragma unroll
            for (int w = 0; w < V; w++)
                if ((uint32_t)w == pt.y) t[w] = (t[w] & ~(pt.w << pt.z)) | (dst << pt.z);
        }
        return;
    }
    // mixed radix, last participant fastest (itertools.product order)
    for (int k = (int)rl.x - 1; k >= 0; k--) {
        const uint4 pt = __ldg(&N.parts[rl.y + k]);
        const uint32_t sq = field_get<V>(s, pt.y, pt.z, pt.w);
        const uint2 l = __ldg(&N.rq[pt.x + sq]);
        uint32_t dig = 0;
        if (l.y > 1) {
            dig = c % l.y;
            c /= l.y;
        }
        const uint32_t dst = __ldg(&N.rdst[l.x + dig]);
#pragma unroll
        for (int w = 0; w < V; w++)
            if ((uint32_t)w == pt.y) t[w] = (t[w] & ~(pt.w << pt.z)) | (dst << pt.z);
    }
}

template <int V, bool EMIT>
__device__ __forceinline__ void process_rules(const NetDesc& N, const uint32_t* s, const uint4 e, uint64_t& count,
                                              uint32_t& n, uint32_t lo, uint32_t hi, uint32_t* out);

// The moves of one process in state s: independent moves from qtab entry
// e, then the rules this process triggers (it is their first participant).
template <int V, bool EMIT>
__device__ __forceinline__ void process_moves(const NetDesc& N, const uint32_t* s, const uint4 pr,
                                              const uint4 e, uint64_t& count, uint32_t& n,
                                              uint32_t lo, uint32_t hi, uint32_t* out) {
    count += e.z;
    if (EMIT && n < hi && n + e.y > lo) {
        for (uint32_t d = 0; d < e.y; d++) {
            const uint32_t idx = n + d;
            if (idx < lo || idx >= hi) continue;
            const uint32_t dst = __ldg(&N.im_dst[e.x + d]);
            uint32_t* o = out + (uint64_t)(idx - lo) * V;
#pragma unroll
            for (int w = 0; w < V; w++)
                o[w] = (uint32_t)w == pr.x ? (s[w] & ~(pr.z << pr.y)) | (dst << pr.y) : s[w];
        }
    }
    n += e.y;
    process_rules<V, EMIT>(N, s, e, count, n, lo, hi, out);
}

// The rules whose first participant is the process with qtab entry e.
template <int V, bool EMIT>
__device__ __forceinline__ void process_rules(const NetDesc& N, const uint32_t* s, const uint4 e, uint64_t& count,
                                              uint32_t& n, uint32_t lo, uint32_t hi, uint32_t* out) {
    uint32_t t[V];
    // packed: the trigger count rides in qtab, so states that trigger no
    // rule (most of them) skip the dependent load of the trigger list
    const uint32_t toff = N.trig_packed ? (e.w & 0xffffffu) : e.w;
    uint32_t nt = N.trig_packed ? (e.w >> 24) : 255u;
    if (nt == 255u) nt = __ldg(&N.trig[toff]);
    for (uint32_t x = 0; x < nt; x++) {
        const uint32_t r = __ldg(&N.trig[toff + 1 + x]);
        const uint4 rl = __ldg(&N.rules[r]);
        uint64_t combos = 1;
        for (uint32_t k = 0; k < rl.x; k++) {
            const uint4 pt = __ldg(&N.parts[rl.y + k]);
            const uint2 l = __ldg(&N.rq[pt.x + field_get<V>(s, pt.y, pt.z, pt.w)]);
            combos *= l.y;
            if (!combos) break;
        }
        if (!combos) continue;
        const uint32_t nd = rl.z ? __ldg(&N.dedup[rl.z]) : 0u;  // offset 0: the empty list
        if (nd == 0) {
            count += combos;
            if (EMIT && n < hi && n + combos > lo) {
                for (uint32_t c = 0; c < (uint32_t)combos; c++) {
                    const uint64_t idx = n + c;
                    if (idx < lo || idx >= hi) continue;
                    rule_target<V>(N, rl, c, s, t);
                    uint32_t* o = out + (uint64_t)(idx - lo) * V;
#pragma unroll
                    for (int w = 0; w < V; w++) o[w] = t[w];
                }
            }
            n += (uint32_t)combos;
        } else {
            for (uint32_t c = 0; c < (uint32_t)combos; c++) {
                rule_target<V>(N, rl, c, s, t);
                bool dup = false;
                for (uint32_t y = 0; y < nd && !dup; y++)
                    dup = rule_generates<V>(N, __ldg(&N.dedup[rl.z + 1 + y]), s, t);
                if (dup) continue;
                count += 1;
                if (EMIT && n >= lo && n < hi) {
                    uint32_t* o = out + (uint64_t)(n - lo) * V;
#pragma unroll
                    for (int w = 0; w < V; w++) o[w] = t[w];
                }
                n++;
            }
        }
    }
}

__device__ __forceinline__ uint4 proc_desc(const NetDesc& N, uint32_t i) {
    return i < GX_PROC_INLINE ? N.proc_c[i] : __ldg(&N.proc[i]);
}

// Expand packed state s.  Returns the number of successor slots n (the
// index space of emitted successors) and the transition count in *count.
// EMIT: successors with index in [lo, hi) are written to out[(idx-lo)*V].
// Independent self-loops are counted but never emitted (t == s is already
// in the table); a rule combination whose (result, target) an earlier rule
// of the same result already produced is neither counted nor emitted
// (network.py:226-230).  (Unrolling the process loop 4x to overlap the qtab
// loads was measured on the B200: 12% slower -- the larger loop body costs
// more than the overlap gains.)
template <int V, bool EMIT>
__device__ __forceinline__ uint32_t expand_state(const NetDesc& N, const uint32_t* s,
                                                 uint64_t* count_out, uint32_t lo, uint32_t hi,
                                                 uint32_t* out) {
    uint64_t count = 0;
    uint32_t n = 0;
    if (N.ngroups) {
        // grouped: one table lookup per process group; its independent
        // successors are s with one word XOR-ed; processes that trigger
        // rules there take the per-process rule path (same successor set
        // and counts as the loop below, network.py:184-238)
        for (uint32_t g = 0; g < N.ngroups; g++) {
            const uint4 gd = N.gdesc[g];
            const uint32_t wsel = gd.x & 0xffu;
            const uint4 e = __ldg(&N.gtab[gd.w + ((word_at<V>(s, wsel) >> gd.y) & gd.z)]);
            count += e.x;
            if (EMIT && n < hi && n + e.y > lo) {
                for (uint32_t d = 0; d < e.y; d++) {
                    const uint32_t idx = n + d;
                    if (idx < lo || idx >= hi) continue;
                    const uint32_t dx = __ldg(&N.gdelta[e.z + d]);
                    uint32_t* o = out + (uint64_t)(idx - lo) * V;
#pragma unroll
                    for (int w = 0; w < V; w++) o[w] = (uint32_t)w == wsel ? s[w] ^ dx : s[w];
                }
            }
            n += e.y;
            for (uint32_t tm = e.w; tm; tm &= tm - 1) {
                const uint32_t p = ((gd.x >> 8) & 0xffffu) + (uint32_t)(__ffs(tm) - 1);
                const uint4 pr = proc_desc(N, p);
                const uint4 qe = __ldg(&N.qtab[pr.w + field_get<V>(s, pr.x, pr.y, pr.z)]);
                process_rules<V, EMIT>(N, s, qe, count, n, lo, hi, out);
            }
        }
        *count_out = count;
        return n;
    }
    for (uint32_t i = 0; i < N.nproc; i++) {
        const uint4 pr = proc_desc(N, i);
        const uint4 e = __ldg(&N.qtab[pr.w + field_get<V>(s, pr.x, pr.y, pr.z)]);
        process_moves<V, EMIT>(N, s, pr, e, count, n, lo, hi, out);
    }
    *count_out = count;
    return n;
}

}  // namespace gx
