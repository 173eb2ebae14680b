// gx_bench.cuh -- keys of the isolated FINDORPUT benchmark, generated on
// the device (the reference's duplication sequence, bench.py:35-96, as a
// keyed bijection: position e -> row min(perm(e) / d, unique - 1) -> key),
// shared by the single-GPU bench (gx_explore.cu) and the hash-partitioned
// multi-GPU one (gx_shard.cu).
#pragma once
#include "gx_device.cuh"

namespace gx {

// bijection on [0, 2^bits), keyed
__device__ __forceinline__ uint64_t perm_bits(uint64_t x, int bits, uint64_t key) {
    const uint64_t mask = bits >= 64 ? ~0ull : ((1ull << bits) - 1);
    const int sh = bits / 2 + 1;
#pragma unroll
    for (int r = 0; r < 4; r++) {
        x = (x * (0x9E3779B97F4A7C15ull | 1ull)) & mask;
        x ^= x >> sh;
        x = (x + (key * (2 * r + 1) ^ (0xD6E8FEB86659FD93ull >> r))) & mask;
        x ^= x >> (sh > 3 ? sh - 2 : 1);
    }
    return x & mask;
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// unique row r -> key words (injective in r for r < 2^(2*kb))
template <int V>
__device__ __forceinline__ void bench_row(uint64_t r, int kb, uint64_t seed, uint32_t* key) {
    const uint64_t m = kb >= 32 ? 0xffffffffull : ((1ull << kb) - 1);
    key[0] = (uint32_t)perm_bits(r & m, kb, seed);
    if (V >= 2) key[1] = (uint32_t)((perm_bits((r >> kb) & m, kb, seed ^ 0x5bd1e995ull) ^ mix64(key[0] + seed)) & m);
#pragma unroll
    for (int w = 2; w < V; w++) key[w] = (uint32_t)(mix64(r * 0x9E3779B97F4A7C15ull + w + seed) & m);
}

struct BenchArgs {
    uint64_t total, dup, unique, row_base, seed;
    int32_t key_bits, perm_bits_n;
    unsigned long long* ctr;  // [0] inserted, [1] full, [2] bucket loads (staged kernel)
};

template <int V>
__device__ __forceinline__ void bench_key(const BenchArgs& B, uint64_t e, uint32_t* key) {
    uint64_t p = e;
    do {
        p = perm_bits(p, B.perm_bits_n, B.seed);
    } while (p >= B.total);
    uint64_t row = p / B.dup;
    if (row >= B.unique) row = B.unique - 1;
    bench_row<V>(row + B.row_base, B.key_bits, B.seed, key);
}

}  // namespace gx
