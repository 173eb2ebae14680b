// gx_internal.h -- host-side structures shared by the libgx translation units.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "../../include/gx.h"
#include "gx_device.cuh"

namespace gx {

void set_error(const char* fmt, ...);
void count_launch(uint64_t n = 1);
int sm_count();

#define GX_CUDA(call)                                                                     \
    do {                                                                                  \
        cudaError_t _e = (call);                                                          \
        if (_e != cudaSuccess) {                                                          \
            ::gx::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), __FILE__, \
                            __LINE__, cudaGetErrorString(_e));                            \
            return GX_EINTERNAL;                                                          \
        }                                                                                 \
    } while (0)

#define GX_LAUNCHED()                   \
    do {                                \
        GX_CUDA(cudaGetLastError());    \
        ::gx::count_launch();           \
    } while (0)

// Device network, network.py:43-62 flattened (see gx.h gx_network_csr).
#define GX_PROC_INLINE 32  // processes whose descriptors ride in the kernel parameters
#define GX_GROUP_INLINE 32  // process groups the grouped expansion supports (else per process)
#ifndef GX_GROUP_BITS
#define GX_GROUP_BITS 10    // joint field bits per group table (2^bits entries of 16 bytes)
#endif

struct NetDesc {
    const uint4* proc;   // {word, shift, mask, qbase}
    const uint4* qtab;   // per (proc, state): {im_off, im_n, im_cnt, trig}; trig =
                         // trig_off | nt << 24 when trig_packed (nt < 255), else trig_off
    const uint32_t* im_dst;
    const uint32_t* trig;   // [n, rule...]
    const uint4* rules;     // {npart, part_off, dedup_off, result}
    const uint4* parts;     // {rq_base, word, shift, mask}
    const uint2* rq;        // {off, n}
    const uint32_t* rdst;
    const uint32_t* dedup;  // [n, rule...]
    const uint4* rmask;     // per rule: participant bits of words 0..3 (vlen <= 4), or null
    uint32_t nproc, nrules, vlen, trig_packed;
    // the first GX_PROC_INLINE process descriptors again, in the parameter
    // (constant) bank: the expansion loop walks them in lockstep across the
    // warp, so a uniform constant load replaces an L1 round trip
    uint4 proc_c[GX_PROC_INLINE];
    // process groups (gx_net_create): runs of consecutive processes whose
    // fields are adjacent in one word, looked up together -- one table
    // entry per joint local-state code gives the group's transition count,
    // independent successors (XOR deltas in gdelta) and which of its
    // processes trigger rules.  ngroups = 0: the per-process loop.
    const uint4* gtab;       // {count, nsucc, delta_off, trigger mask}
    const uint32_t* gdelta;  // independent successors as XOR masks of the group's word
    uint32_t ngroups, pad_g[3];
    uint4 gdesc[GX_GROUP_INLINE];  // {word | p0 << 8 | np << 24, shift, mask, gtab base}
};

// A growable device scratch buffer.
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    int ensure(size_t need) {
        if (need <= bytes) return GX_OK;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        size_t nb = need < 4096 ? 4096 : need;
        GX_CUDA(cudaMalloc(&p, nb));
        bytes = nb;
        return GX_OK;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
};

}  // namespace gx

// Counter cells of a table (device u64[16]).
enum {
    CTR_OCCUPIED = 0,  // slots published
    CTR_OLD = 1,       // slots claimed NEW -> OLD
    CTR_FULL = 2,      // TABLE_FULL results (scratch)
    CTR_SCRATCH = 3,
    CTR_N = 16
};

struct gx_table {
    gx::TableDesc d;
    gx_table_cfg cfg;
    cudaStream_t stream;
    uint64_t total_slots;
    uint64_t* d_ctr;   // CTR_N cells
    uint64_t* h_ctr;   // pinned mirror
    gx::DevBuf keys, codes, handles, aux, aux2, gfilter;
};

struct gx_net {
    gx::NetDesc d;
    cudaStream_t stream;
    uint32_t vlen, nproc;
    std::vector<uint32_t> initial;
    std::vector<uint4> proc_host;  // for unpacking on the host (composite order)
    uint32_t* d_blob;
    uint32_t* d_initial;
    gx::DevBuf scratch;
    gx::DevBuf dl;        // deadlock buffer
    uint64_t dl_recorded; // deadlocks recorded by gx_expand_route (multi-GPU driver)
};

namespace gx {
// table-side helpers used by the explore translation unit
int table_find_or_put_dev(gx_table* t, const uint32_t* d_keys, uint64_t n, uint8_t* d_codes,
                          int64_t* d_handles, int serial, int group);
int table_fixup_status(gx_table* t, const uint32_t* d_new_keys, uint64_t n_new);
// keep the GX_DEADLOCK_KEEP smallest deadlock states (composite order)
void keep_smallest(const gx_net* n, std::vector<uint32_t>& kept, const uint32_t* add, uint64_t cnt);
// the exact deadlocks of frontier F[0, nF) merged into kept, dl_cap states at a time
int rescan_deadlocks(const gx_net* n, const uint32_t* F, uint64_t nF, uint32_t* dl, uint64_t dl_cap,
                     unsigned long long* cell, cudaStream_t st, std::vector<uint32_t>& kept);
}  // namespace gx
