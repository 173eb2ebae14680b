// gx_table.cu -- the B200 state table: creation, batch FINDORPUT, claim,
// scan/compaction, occupancy and inspection (reference: hashtable.py).
#include <algorithm>
#include <atomic>
#include <cstring>
#include <mutex>

#include "gx_internal.h"

namespace gx {

static thread_local char g_err[1024];
static std::atomic<uint64_t> g_launches{0};

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

void count_launch(uint64_t n) { g_launches += n; }

int sm_count() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0)
            sms = 148;
    }
    return sms;
}

static uint64_t splitmix_next(uint64_t* x) {
    *x += 0x9E3779B97F4A7C15ull;
    uint64_t z = *x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ uint32_t warp_sum_u32(uint32_t v) {
    return __reduce_add_sync(FULLMASK, v);
}

__device__ __forceinline__ unsigned long long warp_sum_u64(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULLMASK, v, o);
    return v;
}

// --------------------------------------------------------- FINDORPUT batch

template <int BW, int V, int G>
__global__ void __launch_bounds__(256) k_fop_mark(TableDesc T, const uint32_t* __restrict__ keys,
                                                  uint64_t n, uint8_t* codes, int64_t* handles,
                                                  unsigned long long* ctr, int serial) {
    const int lane = threadIdx.x & 31;
    const int grp = lane / G;
    const bool leader = (lane & (G - 1)) == 0;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nwarps = (gridDim.x * (uint64_t)blockDim.x) >> 5;
    unsigned long long ins = 0, full = 0;
    if (serial) {
        // one key at a time, in order: the reference's single-threaded placement
        for (uint64_t e = warp; e < n; e += nwarps) {
            const bool active = grp == 0;
            uint32_t key[V];
#pragma unroll
            for (int w = 0; w < V; w++) key[w] = keys[e * V + w];
            int64_t hd;
            const int code = probe_mark<BW, V, G>(T, active, key, fold<V>(T.salt, key), &hd);
            if (active && leader) {
                if (codes) codes[e] = (uint8_t)code;
                if (handles) handles[e] = hd;
                ins += code == INSERTED;
                full += code == TABLE_FULL;
            }
        }
    } else {
        using S = ProbeShape<BW, G>;
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
                if (act[u] && leader) {
                    const uint64_t e = base + u * S::R + grp;
                    if (codes) codes[e] = (uint8_t)code[u];
                    if (handles) handles[e] = hd[u];
                    ins += code[u] == INSERTED;
                    full += code[u] == TABLE_FULL;
                }
            }
        }
    }
    ins = warp_sum_u64(ins);
    full = warp_sum_u64(full);
    if (lane == 0) {
        if (ins) atomicAdd(&ctr[CTR_OCCUPIED], ins);
        if (full) atomicAdd(&ctr[CTR_FULL], full);
    }
}

__global__ void __launch_bounds__(256) k_fop_status(TableDesc T, const uint32_t* __restrict__ keys,
                                                    uint64_t n, uint8_t* codes, int64_t* handles,
                                                    unsigned long long* ctr, int serial) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nth = serial ? 1 : gridDim.x * (uint64_t)blockDim.x;
    unsigned long long ins = 0, full = 0;
    uint32_t key[GX_MAXV];
    if (!serial || tid == 0) {
        for (uint64_t e = tid; e < n; e += nth) {
            for (int w = 0; w < (int)T.vlen; w++) key[w] = keys[e * T.vlen + w];
            const uint64_t h = fold_rt(T.salt, key, (int)T.vlen);
            int64_t hd;
            const int code = probe_status(T, key, h, &hd);
            if (codes) codes[e] = (uint8_t)code;
            if (handles) handles[e] = hd;
            ins += code == INSERTED;
            full += code == TABLE_FULL;
        }
    }
    ins = warp_sum_u64(ins);
    full = warp_sum_u64(full);
    if ((threadIdx.x & 31) == 0) {
        if (ins) atomicAdd(&ctr[CTR_OCCUPIED], ins);
        if (full) atomicAdd(&ctr[CTR_FULL], full);
    }
}

typedef void (*fop_kernel_t)(TableDesc, const uint32_t*, uint64_t, uint8_t*, int64_t*,
                             unsigned long long*, int);

template <int BW, int V>
static fop_kernel_t pick_g(int g) {
    switch (g) {
        case 1: return k_fop_mark<BW, V, 1>;
        case 2: if (BW >= 8) return k_fop_mark<BW, V, (BW >= 8 ? 2 : 1)>; break;
        case 4: if (BW >= 16) return k_fop_mark<BW, V, (BW >= 16 ? 4 : 1)>; break;
        case 8: if (BW >= 32) return k_fop_mark<BW, V, (BW >= 32 ? 8 : 1)>; break;
    }
    return nullptr;
}

template <int BW>
static fop_kernel_t pick_v(int v, int g) {
    switch (v) {
        case 1: return pick_g<BW, 1>(g);
        case 2: return pick_g<BW, 2>(g);
        case 4: return (BW >= 4) ? pick_g<BW, 4>(g) : nullptr;
    }
    return nullptr;
}

// default probe group (lanes per bucket), from the round-1 sweep on B200:
// 32-word buckets: 2 lanes x 64 B; smaller buckets: one lane per bucket
int default_group(int bw) { return bw >= 32 ? 2 : (bw >= 16 ? 2 : 1); }

static fop_kernel_t pick_fop(int bw, int v, int g) {
    switch (bw) {
        case 4: return pick_v<4>(v, g);
        case 8: return pick_v<8>(v, g);
        case 16: return pick_v<16>(v, g);
        case 32: return pick_v<32>(v, g);
    }
    return nullptr;
}

static int grid_for(uint64_t items_per_block_round, uint64_t n) {
    uint64_t want = (n + items_per_block_round - 1) / items_per_block_round;
    uint64_t cap = (uint64_t)sm_count() * 8;
    if (want < 1) want = 1;
    return (int)std::min(want, cap);
}

int table_find_or_put_dev(gx_table* t, const uint32_t* d_keys, uint64_t n, uint8_t* d_codes,
                          int64_t* d_handles, int serial, int group) {
    if (n == 0) return GX_OK;
    const TableDesc& T = t->d;
    if (T.mode == MODE_MARK) {
        int g = group > 0 ? group : default_group((int)T.bw);
        fop_kernel_t k = pick_fop((int)T.bw, (int)T.vlen, g);
        if (!k) {
            set_error("no FINDORPUT kernel for bw=%u vlen=%u group=%d", T.bw, T.vlen, g);
            return GX_EINPUT;
        }
        int grid = serial ? 1 : grid_for(256 / g, n);
        k<<<grid, serial ? 32 : 256, 0, t->stream>>>(T, d_keys, n, d_codes, d_handles,
                                                    (unsigned long long*)t->d_ctr, serial);
    } else {
        int grid = serial ? 1 : grid_for(256, n);
        k_fop_status<<<grid, serial ? 32 : 256, 0, t->stream>>>(T, d_keys, n, d_codes, d_handles,
                                                               (unsigned long long*)t->d_ctr, serial);
    }
    GX_LAUNCHED();
    return GX_OK;
}

// ------------------------------------------------------------- slot state

__device__ __forceinline__ uint32_t slot_status_of(const TableDesc& T, uint64_t bucket, int j) {
    uint8_t b = T.status[bucket * (uint64_t)T.stride + j];
    if (T.mode == MODE_STATUS) return b;
    if (!slot_occupied(T, bucket, j)) return EMPTY;
    return b == OLD ? OLD : NEW;
}

__device__ __forceinline__ void read_words(const TableDesc& T, uint64_t bucket, int j, uint32_t* out) {
    const uint32_t* d = T.data + bucket * (uint64_t)T.bw + T.offsets[j];
    for (int w = 0; w < (int)T.vlen; w++) {
        uint32_t x = __ldcg(d + w);
        if (T.mode == MODE_MARK && w == (int)T.mark_word) x &= ~T.mark;
        out[w] = x;
    }
}

// claim_new, hashtable.py:296-313.  In MODE_MARK an occupied slot's status
// byte is 0 while NEW and OLD after the claim.
__global__ void k_claim(TableDesc T, const int64_t* __restrict__ handles, uint64_t n, uint8_t* out,
                        unsigned long long* ctr) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    unsigned long long won = 0;
    if (i < n) {
        const int64_t h = handles[i];
        uint32_t ok = 0;
        if (h >= 0 && (uint64_t)h < T.nb * T.spb) {
            const uint64_t bucket = (uint64_t)h / T.spb;
            const int j = (int)((uint64_t)h % T.spb);
            uint8_t* cell = T.status + bucket * (uint64_t)T.stride + j;
            uint32_t seen;
            if (T.mode == MODE_STATUS)
                ok = status_word_cas_byte(cell, NEW, OLD, &seen);
            else if (slot_occupied(T, bucket, j))
                ok = status_word_cas_byte(cell, 0u, OLD, &seen);
        }
        out[i] = (uint8_t)ok;
        won = ok;
    }
    won = warp_sum_u64(won);
    if ((threadIdx.x & 31) == 0 && won) atomicAdd(&ctr[CTR_OLD], won);
}

// Selection of slots in bucket-major order (scan_new / occupied dump):
// each block owns a contiguous bucket range; pass 1 counts, the host scans
// the block counts, pass 2 writes with a block-wide exclusive scan per
// round of blockDim buckets so the output is globally sorted.
enum { SEL_NEW = 0, SEL_OCCUPIED = 1 };

__device__ __forceinline__ uint32_t select_mask(const TableDesc& T, uint64_t bucket, int pred) {
    uint32_t m = 0;
    for (int j = 0; j < (int)T.spb; j++) {
        uint32_t st = slot_status_of(T, bucket, j);
        bool sel = pred == SEL_NEW ? st == NEW : st >= NEW;
        m |= (sel ? 1u : 0u) << j;
    }
    return m;
}

__global__ void __launch_bounds__(256) k_select_count(TableDesc T, uint64_t first, uint64_t last,
                                                      uint64_t chunk, int pred,
                                                      unsigned long long* blockcounts) {
    const uint64_t lo = first + blockIdx.x * chunk;
    const uint64_t hi = min(last, lo + chunk);
    unsigned long long c = 0;
    for (uint64_t b = lo + threadIdx.x; b < hi; b += blockDim.x) c += __popc(select_mask(T, b, pred));
    c = warp_sum_u64(c);
    __shared__ unsigned long long part[8];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) s += part[w];
        blockcounts[blockIdx.x] = s;
    }
}

__global__ void __launch_bounds__(256) k_select_write(TableDesc T, uint64_t first, uint64_t last,
                                                      uint64_t chunk, int pred,
                                                      const unsigned long long* blockoffs,
                                                      uint64_t cap, int64_t* out_h, uint8_t* out_s,
                                                      uint32_t* out_w) {
    const uint64_t lo = first + blockIdx.x * chunk;
    const uint64_t hi = min(last, lo + chunk);
    __shared__ uint32_t wsum[8];
    __shared__ unsigned long long running;
    if (threadIdx.x == 0) running = blockoffs[blockIdx.x];
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (uint64_t b0 = lo; b0 < hi; b0 += blockDim.x) {
        const uint64_t b = b0 + threadIdx.x;
        const uint32_t m = b < hi ? select_mask(T, b, pred) : 0u;
        const uint32_t c = __popc(m);
        // block exclusive scan of c
        uint32_t x = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            uint32_t y = __shfl_up_sync(FULLMASK, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[wid] = x;
        __syncthreads();
        uint32_t wpre = 0, total = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
            if (w < wid) wpre += wsum[w];
            total += wsum[w];
        }
        unsigned long long pos = running + wpre + x - c;
        uint32_t mm = m;
        while (mm) {
            const int j = __ffs(mm) - 1;
            mm &= mm - 1;
            if (pos < cap) {
                if (out_h) out_h[pos] = (int64_t)(b * T.spb + j);
                if (out_s) out_s[pos] = (uint8_t)slot_status_of(T, b, j);
                if (out_w) read_words(T, b, j, out_w + pos * T.vlen);
            }
            pos++;
        }
        __syncthreads();
        if (threadIdx.x == 0) running += total;
        __syncthreads();
    }
}

static int select_slots(gx_table* t, uint64_t first, uint64_t last, int pred, int64_t* h_out,
                        uint8_t* s_out, uint32_t* w_out, uint64_t cap, uint64_t* count) {
    if (!t->d.status) {
        set_error("table was created without a status array (GX_TABLE_NO_STATUS)");
        return GX_EINPUT;
    }
    const TableDesc& T = t->d;
    if (last > T.nb) last = T.nb;
    if (first >= last) {
        *count = 0;
        return GX_OK;
    }
    const uint64_t nbk = last - first;
    uint64_t nblocks = std::min<uint64_t>((uint64_t)sm_count() * 4, (nbk + 255) / 256);
    if (nblocks < 1) nblocks = 1;
    const uint64_t chunk = (nbk + nblocks - 1) / nblocks;
    nblocks = (nbk + chunk - 1) / chunk;
    int rc = t->aux.ensure(sizeof(unsigned long long) * nblocks);
    if (rc) return rc;
    unsigned long long* d_bc = (unsigned long long*)t->aux.p;
    k_select_count<<<(int)nblocks, 256, 0, t->stream>>>(T, first, last, chunk, pred, d_bc);
    GX_LAUNCHED();
    std::vector<unsigned long long> bc(nblocks);
    GX_CUDA(cudaMemcpyAsync(bc.data(), d_bc, sizeof(unsigned long long) * nblocks,
                            cudaMemcpyDeviceToHost, t->stream));
    GX_CUDA(cudaStreamSynchronize(t->stream));
    unsigned long long total = 0;
    for (uint64_t i = 0; i < nblocks; i++) {
        unsigned long long c = bc[i];
        bc[i] = total;
        total += c;
    }
    *count = total;
    if ((!h_out && !s_out && !w_out) || total == 0) return GX_OK;
    const uint64_t n = std::min<uint64_t>(total, cap);
    GX_CUDA(cudaMemcpyAsync(d_bc, bc.data(), sizeof(unsigned long long) * nblocks,
                            cudaMemcpyHostToDevice, t->stream));
    rc = t->handles.ensure(sizeof(int64_t) * n);
    if (rc) return rc;
    rc = t->codes.ensure(n);
    if (rc) return rc;
    rc = t->keys.ensure(sizeof(uint32_t) * n * T.vlen);
    if (rc) return rc;
    k_select_write<<<(int)nblocks, 256, 0, t->stream>>>(
        T, first, last, chunk, pred, d_bc, n, h_out ? (int64_t*)t->handles.p : nullptr,
        s_out ? (uint8_t*)t->codes.p : nullptr, w_out ? (uint32_t*)t->keys.p : nullptr);
    GX_LAUNCHED();
    if (h_out)
        GX_CUDA(cudaMemcpyAsync(h_out, t->handles.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost,
                                t->stream));
    if (s_out) GX_CUDA(cudaMemcpyAsync(s_out, t->codes.p, n, cudaMemcpyDeviceToHost, t->stream));
    if (w_out)
        GX_CUDA(cudaMemcpyAsync(w_out, t->keys.p, sizeof(uint32_t) * n * T.vlen,
                                cudaMemcpyDeviceToHost, t->stream));
    GX_CUDA(cudaStreamSynchronize(t->stream));
    return GX_OK;
}

__global__ void k_read_slots(TableDesc T, const int64_t* __restrict__ handles, uint64_t n,
                             uint8_t* st, uint32_t* words) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t h = handles[i];
    if (h < 0 || (uint64_t)h >= T.nb * T.spb) {
        if (st) st[i] = 0xff;
        return;
    }
    const uint64_t bucket = (uint64_t)h / T.spb;
    const int j = (int)((uint64_t)h % T.spb);
    if (st) st[i] = (uint8_t)slot_status_of(T, bucket, j);
    if (words) read_words(T, bucket, j, words + i * T.vlen);
}

// explore epilogue: every occupied slot OLD ...
__global__ void k_mark_all_old(TableDesc T) {
    const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < T.nb; b += stride) {
        for (int j = 0; j < (int)T.spb; j++) {
            if (slot_occupied(T, b, j)) T.status[b * (uint64_t)T.stride + j] = OLD;
        }
    }
}

// ... then the given handles NEW again
__global__ void k_mark_new(TableDesc T, const int64_t* __restrict__ handles, uint64_t n) {
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t h = handles[i];
    if (h < 0) return;
    const uint64_t bucket = (uint64_t)h / T.spb;
    const int j = (int)((uint64_t)h % T.spb);
    T.status[bucket * (uint64_t)T.stride + j] = T.mode == MODE_STATUS ? NEW : 0;
}

// ----------------------------------------------------------- set digest
// Order-independent digest of the occupied slots (include/gx.h
// gx_table_digest): per state the hash of its first `words` words (mark bit
// cleared), summed mod 2^64 and xor-ed, plus the count.  The same function
// is restated in oracle/gx_oracle.c (or_state_hash) and statevec.py.
__device__ __forceinline__ uint64_t dg_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

__device__ __forceinline__ void digest_flush(unsigned long long c, unsigned long long s,
                                             unsigned long long x, unsigned long long* out) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        c += __shfl_xor_sync(FULLMASK, c, o);
        s += __shfl_xor_sync(FULLMASK, s, o);
        x ^= __shfl_xor_sync(FULLMASK, x, o);
    }
    if ((threadIdx.x & 31) == 0 && c) {
        atomicAdd(&out[0], c);
        atomicAdd(&out[1], s);
        atomicXor(&out[2], x);
    }
}

// in-band tables (slot j at word j*V): one thread per 16-byte chunk, a
// streaming pass over the data array
template <int V>
__global__ void __launch_bounds__(256) k_digest_mark(TableDesc T, int words, unsigned long long* out) {
    const uint64_t chunks = T.nb * (uint64_t)T.bw / 4;
    const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
    unsigned long long c = 0, s = 0, x = 0;
    const uint4* d = reinterpret_cast<const uint4*>(T.data);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < chunks; i += stride) {
        const uint4 q = __ldcs(d + i);
        const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (int t = 0; t < 4 / V; t++) {
            if ((w4[t * V + T.mark_word] & T.mark) == 0u) continue;
            uint64_t h = 0x6A09E667F3BCC908ull ^ (uint64_t)words;
            for (int w = 0; w < words; w++) {
                uint32_t y = w4[t * V + w];
                if (w == (int)T.mark_word) y &= ~T.mark;
                h = dg_mix(h ^ (uint64_t)y);
            }
            c++;
            s += h;
            x ^= h;
        }
    }
    digest_flush(c, s, x, out);
}

// any table: one thread per bucket, slots through the status protocol
__global__ void __launch_bounds__(256) k_digest_any(TableDesc T, int words, unsigned long long* out) {
    const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
    unsigned long long c = 0, s = 0, x = 0;
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < T.nb; b += stride) {
        for (int j = 0; j < (int)T.spb; j++) {
            if (!slot_occupied(T, b, j)) continue;
            uint32_t key[GX_MAXV];
            read_words(T, b, j, key);
            uint64_t h = 0x6A09E667F3BCC908ull ^ (uint64_t)words;
            for (int w = 0; w < words; w++) h = dg_mix(h ^ (uint64_t)key[w]);
            c++;
            s += h;
            x ^= h;
        }
    }
    digest_flush(c, s, x, out);
}

// ------------------------------------------------------ sorted dump
// The canonical state dump (statevec.py:93-100: packed words, sorted
// lexicographically) produced on the device: gather the occupied slots'
// first `words` words, then a stable LSD radix sort over the words from
// last to first (8-bit digits, a permutation carried along), then one
// gather in sorted order.  Works on tables without a status array.
constexpr int DS_TILE = 1 << 15;  // elements per radix tile

__global__ void __launch_bounds__(256) k_gather_occupied(TableDesc T, int words, uint32_t* out,
                                                         unsigned long long* ctr, uint64_t cap) {
    const uint64_t stride = gridDim.x * (uint64_t)blockDim.x;
    const int lane = threadIdx.x & 31;
    const uint64_t nb_round = (T.nb + stride - 1) / stride * stride;
    for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nb_round; b += stride) {
        uint32_t occ = 0;
        if (b < T.nb)
            for (int j = 0; j < (int)T.spb; j++) occ |= (slot_occupied(T, b, j) ? 1u : 0u) << j;
        const uint32_t c = __popc(occ);
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(FULLMASK, incl, o);
            if (lane >= o) incl += y;
        }
        unsigned long long base = 0;
        if (lane == 31 && incl) base = atomicAdd(ctr, (unsigned long long)incl);
        base = __shfl_sync(FULLMASK, base, 31) + incl - c;
        for (int j = 0; occ; j++, occ >>= 1) {
            if (!(occ & 1u)) continue;
            if (base < cap) {
                uint32_t key[GX_MAXV];
                read_words(T, b, j, key);
                for (int w = 0; w < words; w++) out[base * words + w] = key[w];
            }
            base++;
        }
    }
}

__global__ void k_iota(uint32_t* perm, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (uint64_t)blockDim.x)
        perm[i] = (uint32_t)i;
}

__global__ void k_word_of(const uint32_t* rows, int words, int w, const uint32_t* perm, uint32_t* key, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (uint64_t)blockDim.x)
        key[i] = rows[(uint64_t)perm[i] * words + w];
}

// per tile: histogram of digit (key >> shift) & 255 -> hist[digit * tiles + tile]
__global__ void __launch_bounds__(256) k_radix_hist(const uint32_t* key, uint64_t n, int shift, uint32_t* hist,
                                                   uint32_t tiles) {
    __shared__ uint32_t h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t lo = (uint64_t)blockIdx.x * DS_TILE, hi = min(n, lo + DS_TILE);
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(&h[(key[i] >> shift) & 255u], 1u);
    __syncthreads();
    hist[threadIdx.x * (uint64_t)tiles + blockIdx.x] = h[threadIdx.x];
}

// exclusive scan of hist[0, m) in place, one block (m is a few million)
__global__ void __launch_bounds__(1024) k_scan_one(uint32_t* a, uint64_t m) {
    __shared__ uint32_t part[1024];
    const uint64_t per = (m + 1023) / 1024;
    const uint64_t lo = threadIdx.x * per, hi = min(m, lo + per);
    uint32_t sum = 0;
    for (uint64_t i = lo; i < hi; i++) sum += a[i];
    part[threadIdx.x] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t run = 0;
        for (int i = 0; i < 1024; i++) {
            const uint32_t x = part[i];
            part[i] = run;
            run += x;
        }
    }
    __syncthreads();
    uint32_t run = part[threadIdx.x];
    for (uint64_t i = lo; i < hi; i++) {
        const uint32_t x = a[i];
        a[i] = run;
        run += x;
    }
}

// stable scatter of one tile by one warp, 32 elements at a time in order
__global__ void __launch_bounds__(32) k_radix_scatter(const uint32_t* key, const uint32_t* perm, uint64_t n,
                                                      int shift, const uint32_t* offs, uint32_t tiles,
                                                      uint32_t* key2, uint32_t* perm2) {
    __shared__ uint32_t cur[256];
    const int lane = threadIdx.x;
    for (int d = lane; d < 256; d += 32) cur[d] = offs[d * (uint64_t)tiles + blockIdx.x];
    __syncwarp();
    const uint64_t lo = (uint64_t)blockIdx.x * DS_TILE, hi = min(n, lo + DS_TILE);
    for (uint64_t b = lo; b < hi; b += 32) {
        const uint64_t i = b + lane;
        const bool a = i < hi;
        const uint32_t k = a ? key[i] : 0u, p = a ? perm[i] : 0u;
        const uint32_t d = a ? (k >> shift) & 255u : 256u;
        const uint32_t grp = __match_any_sync(FULLMASK, d);
        uint32_t lt;
        asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
        const uint32_t pos = a ? cur[d] + __popc(grp & lt) : 0u;
        __syncwarp();
        if (a && (grp & lt) == 0) cur[d] += __popc(grp);
        __syncwarp();
        if (a) {
            key2[pos] = k;
            perm2[pos] = p;
        }
    }
}

__global__ void k_gather_rows(const uint32_t* rows, int words, const uint32_t* perm, uint32_t* out, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += gridDim.x * (uint64_t)blockDim.x)
        for (int w = 0; w < words; w++) out[i * words + w] = rows[(uint64_t)perm[i] * words + w];
}

int table_fixup_status(gx_table* t, const uint32_t* d_new_keys, uint64_t n_new) {
    if (!t->d.status) return GX_OK;  // exploration-only table: no statuses to keep
    const TableDesc& T = t->d;
    int grid = (int)std::min<uint64_t>((uint64_t)sm_count() * 8, (T.nb + 255) / 256);
    if (grid < 1) grid = 1;
    k_mark_all_old<<<grid, 256, 0, t->stream>>>(T);
    GX_LAUNCHED();
    if (n_new) {
        int rc = t->handles.ensure(sizeof(int64_t) * n_new);
        if (rc) return rc;
        // the keys are present: FINDORPUT returns FOUND with their handles
        unsigned long long saved[CTR_N];
        GX_CUDA(cudaMemcpyAsync(saved, t->d_ctr, sizeof saved, cudaMemcpyDeviceToHost, t->stream));
        GX_CUDA(cudaStreamSynchronize(t->stream));
        rc = table_find_or_put_dev(t, d_new_keys, n_new, nullptr, (int64_t*)t->handles.p, 0, 0);
        if (rc) return rc;
        k_mark_new<<<(int)((n_new + 255) / 256), 256, 0, t->stream>>>(T, (const int64_t*)t->handles.p,
                                                                      n_new);
        GX_LAUNCHED();
        GX_CUDA(cudaMemcpyAsync(t->d_ctr, saved, sizeof saved, cudaMemcpyHostToDevice, t->stream));
    }
    return GX_OK;
}

}  // namespace gx

using namespace gx;

// ===================================================================== C ABI

extern "C" {

const char* gx_last_error(void) { return g_err; }

uint64_t gx_kernel_launches(void) { return g_launches.load(); }

int gx_device_info(int32_t* sms, uint64_t* free_b, uint64_t* total_b) {
    size_t f = 0, tt = 0;
    GX_CUDA(cudaMemGetInfo(&f, &tt));
    if (sms) *sms = sm_count();
    if (free_b) *free_b = f;
    if (total_b) *total_b = tt;
    return GX_OK;
}

int gx_sync(void* stream) {
    GX_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    return GX_OK;
}

// slots_per_bucket, hashtable.py:89-111
static int spb_of(int bw, int vlen, int layout) {
    if (bw <= 0 || vlen <= 0) {
        set_error("bucket_words and vector_length must be positive");
        return 0;
    }
    int c;
    if (layout == GX_LAYOUT_HALF) {
        if (bw % 2) {
            set_error("half-bucket layout requires an even bucket size");
            return 0;
        }
        c = 2 * ((bw / 2) / vlen);
    } else if (layout == GX_LAYOUT_PLAIN) {
        c = bw / vlen;
    } else {
        set_error("unknown layout %d", layout);
        return 0;
    }
    if (c == 0) {
        set_error("vector too long for bucket: %d words in a %d-word bucket (%s)", vlen, bw,
                  layout == GX_LAYOUT_HALF ? "half" : "plain");
        return 0;
    }
    return c;
}

int gx_table_create(const gx_table_cfg* cfg, void* stream, gx_table** out) {
    *out = nullptr;
    const int bw = cfg->bucket_words;
    if (bw != 4 && bw != 8 && bw != 16 && bw != 32) {
        set_error("bucket_words must be one of (4, 8, 16, 32), got %d", bw);
        return GX_EINPUT;
    }
    if (cfg->num_hash_functions < 1) {
        set_error("need at least one hash function");
        return GX_EINPUT;
    }
    if (cfg->num_hash_functions > GX_MAXK) {
        set_error("at most %d hash functions are supported, got %d", GX_MAXK, cfg->num_hash_functions);
        return GX_EINPUT;
    }
    if (cfg->vector_length < 1 || cfg->vector_length > GX_MAXV) {
        set_error("vector_length must be in 1..%d, got %d", GX_MAXV, cfg->vector_length);
        return GX_EINPUT;
    }
    const int spb = spb_of(bw, cfg->vector_length, cfg->layout);
    if (!spb) return GX_EINPUT;
    const uint64_t nb = cfg->capacity_words / (uint64_t)bw;
    if (nb < (uint64_t)cfg->num_hash_functions) {
        set_error("capacity_words %llu gives %llu buckets, fewer than %d hash functions",
                  (unsigned long long)cfg->capacity_words, (unsigned long long)nb,
                  cfg->num_hash_functions);
        return GX_EINPUT;
    }
    gx_table* t = new gx_table();
    t->cfg = *cfg;
    t->stream = (cudaStream_t)stream;
    TableDesc& T = t->d;
    memset(&T, 0, sizeof T);
    T.nb = nb;
    T.nb_magic = nb == 1 ? 0 : (uint64_t)(((unsigned __int128)1 << 64) / nb);
    T.bw = (uint32_t)bw;
    T.vlen = (uint32_t)cfg->vector_length;
    T.spb = (uint32_t)spb;
    T.stride = (uint32_t)((spb + 7) & ~7);
    T.k = (uint32_t)cfg->num_hash_functions;
    const int v = cfg->vector_length;
    bool contiguous = true;
    for (int j = 0; j < spb; j++) {
        int off = (cfg->layout == GX_LAYOUT_HALF && j >= spb / 2) ? bw / 2 + (j - spb / 2) * v : j * v;
        T.offsets[j] = (uint8_t)off;
        if (off != j * v) contiguous = false;
    }
    const bool mark_ok = cfg->mark_word >= 0 && cfg->mark_word < v && cfg->mark_bit >= 0 &&
                         cfg->mark_bit < 32 && (v == 1 || v == 2 || v == 4) && contiguous &&
                         spb * v == bw;
    T.mode = mark_ok ? MODE_MARK : MODE_STATUS;
    T.mark_word = mark_ok ? (uint32_t)cfg->mark_word : 0;
    T.mark = mark_ok ? (1u << cfg->mark_bit) : 0;
    uint64_t x = cfg->seed;
    for (int i = 0; i < cfg->num_hash_functions; i++) {
        T.a[i] = splitmix_next(&x) | 1ull;
        T.b[i] = splitmix_next(&x);
    }
    uint64_t y = cfg->seed ^ 0xA5A5A5A5A5A5A5A5ull;
    T.salt = splitmix_next(&y);
    t->total_slots = nb * (uint64_t)spb;
    cudaError_t e1 = cudaMalloc(&T.data, nb * (uint64_t)bw * 4);
    const bool no_status = mark_ok && (cfg->flags & GX_TABLE_NO_STATUS);
    cudaError_t e2 = e1 == cudaSuccess && !no_status ? cudaMalloc(&T.status, nb * (uint64_t)T.stride) : e1;
    cudaError_t e3 = e2 == cudaSuccess ? cudaMalloc(&t->d_ctr, sizeof(uint64_t) * CTR_N) : e2;
    cudaError_t e4 = e3 == cudaSuccess ? cudaMallocHost(&t->h_ctr, sizeof(uint64_t) * CTR_N) : e3;
    if (e4 != cudaSuccess) {
        set_error("device allocation of a %llu-byte table failed: %s",
                  (unsigned long long)(nb * (uint64_t)bw * 4 + nb * (uint64_t)T.stride),
                  cudaGetErrorString(e4));
        cudaGetLastError();
        if (T.data) cudaFree(T.data);
        if (T.status) cudaFree(T.status);
        if (t->d_ctr) cudaFree(t->d_ctr);
        delete t;
        return GX_EINPUT;
    }
    int rc = gx_table_clear(t);
    if (rc) {
        gx_table_destroy(t);
        return rc;
    }
    *out = t;
    return GX_OK;
}

int gx_table_destroy(gx_table* t) {
    if (!t) return GX_OK;
    cudaStreamSynchronize(t->stream);
    cudaFree(t->d.data);
    cudaFree(t->d.status);
    cudaFree(t->d_ctr);
    cudaFreeHost(t->h_ctr);
    t->keys.release();
    t->codes.release();
    t->handles.release();
    t->aux.release();
    t->aux2.release();
    t->gfilter.release();
    delete t;
    return GX_OK;
}

int gx_table_clear(gx_table* t) {
    const TableDesc& T = t->d;
    GX_CUDA(cudaMemsetAsync(T.data, 0, T.nb * (uint64_t)T.bw * 4, t->stream));
    if (T.status) GX_CUDA(cudaMemsetAsync(T.status, 0, T.nb * (uint64_t)T.stride, t->stream));
    GX_CUDA(cudaMemsetAsync(t->d_ctr, 0, sizeof(uint64_t) * CTR_N, t->stream));
    return GX_OK;
}

int gx_table_geometry(const gx_table* t, uint64_t* nb, int32_t* spb, uint64_t* ts) {
    if (nb) *nb = t->d.nb;
    if (spb) *spb = (int32_t)t->d.spb;
    if (ts) *ts = t->total_slots;
    return GX_OK;
}

int gx_table_hash_constants(const gx_table* t, uint64_t* a, uint64_t* b, uint64_t* salt) {
    for (uint32_t i = 0; i < t->d.k; i++) {
        if (a) a[i] = t->d.a[i];
        if (b) b[i] = t->d.b[i];
    }
    if (salt) *salt = t->d.salt;
    return GX_OK;
}

int gx_table_mode(const gx_table* t) { return (int)t->d.mode; }

int gx_find_or_put(gx_table* t, const uint32_t* keys, uint64_t n, uint8_t* codes, int64_t* handles,
                   int32_t serial) {
    if (n == 0) return GX_OK;
    const uint64_t v = t->d.vlen;
    int rc = t->keys.ensure(sizeof(uint32_t) * n * v);
    if (!rc) rc = t->codes.ensure(n);
    if (!rc) rc = t->handles.ensure(sizeof(int64_t) * n);
    if (rc) return rc;
    GX_CUDA(cudaMemcpyAsync(t->keys.p, keys, sizeof(uint32_t) * n * v, cudaMemcpyHostToDevice,
                            t->stream));
    rc = table_find_or_put_dev(t, (const uint32_t*)t->keys.p, n, (uint8_t*)t->codes.p,
                               (int64_t*)t->handles.p, serial, 0);
    if (rc) return rc;
    if (codes) GX_CUDA(cudaMemcpyAsync(codes, t->codes.p, n, cudaMemcpyDeviceToHost, t->stream));
    if (handles)
        GX_CUDA(cudaMemcpyAsync(handles, t->handles.p, sizeof(int64_t) * n, cudaMemcpyDeviceToHost,
                                t->stream));
    GX_CUDA(cudaStreamSynchronize(t->stream));
    return GX_OK;
}

int gx_find_or_put_timed(gx_table* t, const uint32_t* keys, uint64_t n, uint8_t* codes, double* kernel_ms) {
    if (kernel_ms) *kernel_ms = 0.0;
    if (n == 0) return GX_OK;
    const uint64_t v = t->d.vlen;
    int rc = t->keys.ensure(sizeof(uint32_t) * n * v);
    if (!rc) rc = t->codes.ensure(n);
    if (rc) return rc;
    GX_CUDA(cudaMemcpyAsync(t->keys.p, keys, sizeof(uint32_t) * n * v, cudaMemcpyHostToDevice, t->stream));
    cudaEvent_t e0, e1;
    GX_CUDA(cudaEventCreate(&e0));
    GX_CUDA(cudaEventCreate(&e1));
    GX_CUDA(cudaEventRecord(e0, t->stream));
    rc = table_find_or_put_dev(t, (const uint32_t*)t->keys.p, n, (uint8_t*)t->codes.p, nullptr, 0, 0);
    GX_CUDA(cudaEventRecord(e1, t->stream));
    if (codes) GX_CUDA(cudaMemcpyAsync(codes, t->codes.p, n, cudaMemcpyDeviceToHost, t->stream));
    GX_CUDA(cudaStreamSynchronize(t->stream));
    float ms = 0;
    GX_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (rc) return rc;
    if (kernel_ms) *kernel_ms = ms;
    return GX_OK;
}

int gx_find_or_put_device(gx_table* t, const uint32_t* d_keys, uint64_t n, uint8_t* d_codes,
                          int64_t* d_handles, uint64_t* inserted, uint64_t* full) {
    unsigned long long before[CTR_N];
    if (inserted || full) {
        GX_CUDA(cudaMemcpyAsync(before, t->d_ctr, sizeof before, cudaMemcpyDeviceToHost, t->stream));
    }
    int rc = table_find_or_put_dev(t, d_keys, n, d_codes, d_handles, 0, 0);
    if (rc) return rc;
    if (inserted || full) {
        GX_CUDA(cudaMemcpyAsync(t->h_ctr, t->d_ctr, sizeof(uint64_t) * CTR_N, cudaMemcpyDeviceToHost,
                                t->stream));
        GX_CUDA(cudaStreamSynchronize(t->stream));
        if (inserted) *inserted = t->h_ctr[CTR_OCCUPIED] - before[CTR_OCCUPIED];
        if (full) *full = t->h_ctr[CTR_FULL] - before[CTR_FULL];
    }
    return GX_OK;
}

int gx_claim_new(gx_table* t, const int64_t* handles, uint64_t n, uint8_t* claimed) {
    if (!t->d.status) {
        set_error("table was created without a status array (GX_TABLE_NO_STATUS)");
        return GX_EINPUT;
    }
    if (n == 0) return GX_OK;
    int rc = t->handles.ensure(sizeof(int64_t) * n);
    if (!rc) rc = t->codes.ensure(n);
    if (rc) return rc;
    GX_CUDA(cudaMemcpyAsync(t->handles.p, handles, sizeof(int64_t) * n, cudaMemcpyHostToDevice,
                            t->stream));
    k_claim<<<(int)((n + 255) / 256), 256, 0, t->stream>>>(t->d, (const int64_t*)t->handles.p, n,
                                                          (uint8_t*)t->codes.p,
                                                          (unsigned long long*)t->d_ctr);
    GX_LAUNCHED();
    GX_CUDA(cudaMemcpyAsync(claimed, t->codes.p, n, cudaMemcpyDeviceToHost, t->stream));
    GX_CUDA(cudaStreamSynchronize(t->stream));
    return GX_OK;
}

int gx_scan_new(gx_table* t, uint64_t first, uint64_t last, int64_t* out, uint64_t cap,
                uint64_t* count) {
    return select_slots(t, first, last, SEL_NEW, out, nullptr, nullptr, out ? cap : 0, count);
}

int gx_occupancy(gx_table* t, uint64_t* occupied, uint64_t* new_count) {
    GX_CUDA(cudaMemcpyAsync(t->h_ctr, t->d_ctr, sizeof(uint64_t) * CTR_N, cudaMemcpyDeviceToHost,
                            t->stream));
    GX_CUDA(cudaStreamSynchronize(t->stream));
    if (occupied) *occupied = t->h_ctr[CTR_OCCUPIED];
    if (new_count) *new_count = t->h_ctr[CTR_OCCUPIED] - t->h_ctr[CTR_OLD];
    return GX_OK;
}

int gx_read_slots(gx_table* t, const int64_t* handles, uint64_t n, uint8_t* status, uint32_t* words) {
    if (status && !t->d.status) {
        set_error("table was created without a status array (GX_TABLE_NO_STATUS)");
        return GX_EINPUT;
    }
    if (n == 0) return GX_OK;
    const uint64_t v = t->d.vlen;
    int rc = t->handles.ensure(sizeof(int64_t) * n);
    if (!rc) rc = t->codes.ensure(n);
    if (!rc) rc = t->keys.ensure(sizeof(uint32_t) * n * v);
    if (rc) return rc;
    GX_CUDA(cudaMemcpyAsync(t->handles.p, handles, sizeof(int64_t) * n, cudaMemcpyHostToDevice,
                            t->stream));
    k_read_slots<<<(int)((n + 255) / 256), 256, 0, t->stream>>>(
        t->d, (const int64_t*)t->handles.p, n, (uint8_t*)t->codes.p, (uint32_t*)t->keys.p);
    GX_LAUNCHED();
    if (status) GX_CUDA(cudaMemcpyAsync(status, t->codes.p, n, cudaMemcpyDeviceToHost, t->stream));
    if (words)
        GX_CUDA(cudaMemcpyAsync(words, t->keys.p, sizeof(uint32_t) * n * v, cudaMemcpyDeviceToHost,
                                t->stream));
    GX_CUDA(cudaStreamSynchronize(t->stream));
    return GX_OK;
}

int gx_dump(gx_table* t, int64_t* handles, uint8_t* status, uint32_t* words, uint64_t cap,
            uint64_t* count) {
    return select_slots(t, 0, t->d.nb, SEL_OCCUPIED, handles, status, words, cap, count);
}

int gx_dump_sorted(gx_table* t, int32_t words, uint32_t* out, uint64_t capacity, uint64_t* count) {
    const TableDesc& T = t->d;
    if (words < 1 || words > (int32_t)T.vlen) {
        set_error("sorted dump over %d words of a %u-word table", words, T.vlen);
        return GX_EINPUT;
    }
    cudaStream_t st = t->stream;
    unsigned long long* c = (unsigned long long*)t->d_ctr + CTR_SCRATCH;
    // count first
    GX_CUDA(cudaMemsetAsync(c, 0, 8, st));
    const int grid = sm_count() * 8;
    k_gather_occupied<<<grid, 256, 0, st>>>(T, words, nullptr, c, 0);
    GX_LAUNCHED();
    unsigned long long n = 0;
    GX_CUDA(cudaMemcpyAsync(&n, c, 8, cudaMemcpyDeviceToHost, st));
    GX_CUDA(cudaStreamSynchronize(st));
    *count = n;
    if (!out || n == 0) return GX_OK;
    if (n > 0xffffffffull) {
        set_error("sorted dump of %llu states exceeds the 32-bit permutation", n);
        return GX_EINPUT;
    }
    const uint32_t tiles = (uint32_t)((n + DS_TILE - 1) / DS_TILE);
    // rows | key | key2 | perm | perm2 | hist
    const uint64_t b_rows = 4 * n * words, b_vec = 4 * n, b_hist = 4ull * 256 * tiles;
    DevBuf buf;
    int rc = buf.ensure(b_rows + 4 * b_vec + b_hist + 64);
    if (rc) return rc;
    uint32_t* rows = (uint32_t*)buf.p;
    uint32_t* key = rows + n * words;
    uint32_t* key2 = key + n;
    uint32_t* perm = key2 + n;
    uint32_t* perm2 = perm + n;
    uint32_t* hist = perm2 + n;
    GX_CUDA(cudaMemsetAsync(c, 0, 8, st));
    k_gather_occupied<<<grid, 256, 0, st>>>(T, words, rows, c, n);
    GX_LAUNCHED();
    k_iota<<<grid, 256, 0, st>>>(perm, n);
    GX_LAUNCHED();
    for (int w = words - 1; w >= 0; w--) {
        k_word_of<<<grid, 256, 0, st>>>(rows, words, w, perm, key, n);
        GX_LAUNCHED();
        for (int shift = 0; shift < 32; shift += 8) {
            k_radix_hist<<<tiles, 256, 0, st>>>(key, n, shift, hist, tiles);
            GX_LAUNCHED();
            k_scan_one<<<1, 1024, 0, st>>>(hist, 256ull * tiles);
            GX_LAUNCHED();
            k_radix_scatter<<<tiles, 32, 0, st>>>(key, perm, n, shift, hist, tiles, key2, perm2);
            GX_LAUNCHED();
            std::swap(key, key2);
            std::swap(perm, perm2);
        }
    }
    const uint64_t m = std::min<uint64_t>(n, capacity);
    uint32_t* sorted = key2;  // free scratch of n words ... reuse rows-sized space below
    DevBuf outb;
    rc = outb.ensure(4 * n * words);
    if (rc) {
        buf.release();
        return rc;
    }
    sorted = (uint32_t*)outb.p;
    k_gather_rows<<<grid, 256, 0, st>>>(rows, words, perm, sorted, n);
    GX_LAUNCHED();
    GX_CUDA(cudaMemcpyAsync(out, sorted, 4 * m * words, cudaMemcpyDeviceToHost, st));
    GX_CUDA(cudaStreamSynchronize(st));
    buf.release();
    outb.release();
    return GX_OK;
}

int gx_table_digest(gx_table* t, int32_t words, uint64_t* out) {
    const TableDesc& T = t->d;
    if (words < 1 || words > (int32_t)T.vlen) {
        set_error("digest over %d words of a %u-word table", words, T.vlen);
        return GX_EINPUT;
    }
    unsigned long long* c = (unsigned long long*)t->d_ctr + CTR_SCRATCH;  // cells 3..5
    GX_CUDA(cudaMemsetAsync(c, 0, 3 * sizeof(unsigned long long), t->stream));
    const int grid = sm_count() * 8;
    const bool inband = T.mode == MODE_MARK && (T.vlen == 1 || T.vlen == 2 || T.vlen == 4);
    if (inband && T.vlen == 1)
        k_digest_mark<1><<<grid, 256, 0, t->stream>>>(T, words, c);
    else if (inband && T.vlen == 2)
        k_digest_mark<2><<<grid, 256, 0, t->stream>>>(T, words, c);
    else if (inband)
        k_digest_mark<4><<<grid, 256, 0, t->stream>>>(T, words, c);
    else
        k_digest_any<<<grid, 256, 0, t->stream>>>(T, words, c);
    GX_LAUNCHED();
    GX_CUDA(cudaMemcpyAsync(out, c, 3 * sizeof(uint64_t), cudaMemcpyDeviceToHost, t->stream));
    GX_CUDA(cudaStreamSynchronize(t->stream));
    return GX_OK;
}

}  // extern "C"
