// gx_micro.cu -- the random-access HBM roofline R(g):
// aligned random reads of g bytes (g = 16/32/64/128, the bucket sizes of
// bw 4/8/16/32) over a buffer far larger than L2, plus the same pattern
// with a 64-bit CAS on every access (the FINDORPUT insert path).  This is
// the denominator the hash-table probes are judged against: a probe can
// never beat the rate at which HBM serves random g-byte segments.
#include <cuda.h>

#include "gx_internal.h"

namespace gx {

__device__ __forceinline__ uint64_t rmix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// G lanes per segment (G = g / 16), each a 16-byte load; every lane group
// keeps UNR segments in flight.  `segments` = buffer bytes / g.
template <int G, int UNR, bool CAS>
__global__ void __launch_bounds__(256) k_random_read(const uint4* __restrict__ buf, uint64_t segments,
                                                     uint64_t groups_total, uint64_t seed,
                                                     unsigned long long* sink) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t grp = tid / G;
    const int gl = (int)(tid % G);
    const uint64_t ngrp = (gridDim.x * (uint64_t)blockDim.x) / G;
    uint32_t acc = 0;
    for (uint64_t base = grp * UNR; base < groups_total; base += ngrp * UNR) {
        uint4 v[UNR];
        uint64_t seg[UNR];
#pragma unroll
        for (int u = 0; u < UNR; u++) {
            seg[u] = __umul64hi(rmix(seed + base + u), segments);
            v[u] = __ldcg(buf + seg[u] * G + gl);
        }
#pragma unroll
        for (int u = 0; u < UNR; u++) {
            acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
            if (CAS && gl == 0 && (v[u].x | v[u].y) == 0u) {
                // the insert path: claim the segment's first 8 bytes (only
                // when empty, as FINDORPUT does); the buffer is zeroed once
                unsigned long long* p = (unsigned long long*)(buf + seg[u] * G);
                atomicCAS(p, 0ull, 0x8000000000000000ull | (seg[u] + 1));
            }
        }
    }
    if (acc == 0x9E3779B9u) atomicAdd(sink, 1ull);  // keep the loads alive
}

typedef void (*rr_kernel_t)(const uint4*, uint64_t, uint64_t, uint64_t, unsigned long long*);

template <bool CAS>
static rr_kernel_t pick_rr(int g) {
    switch (g) {
        case 16: return k_random_read<1, 8, CAS>;
        case 32: return k_random_read<2, 8, CAS>;
        case 64: return k_random_read<4, 8, CAS>;
        case 128: return k_random_read<8, 8, CAS>;
    }
    return nullptr;
}

}  // namespace gx

using namespace gx;

extern "C" int gx_random_access_bench_alloc(uint64_t, int32_t, uint64_t, int32_t, int32_t, int32_t,
                                            double*, double*, uint64_t*);

// Driver-API entry points resolved through the runtime (no link-time
// dependency on libcuda, so the library still loads on a CPU-only host).
struct DrvVmm {
    CUresult (*granularity)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);
    CUresult (*reserve)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
    CUresult (*create)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*, unsigned long long);
    CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
    CUresult (*access)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
    CUresult (*unmap)(CUdeviceptr, size_t);
    CUresult (*release)(CUmemGenericAllocationHandle);
    CUresult (*addr_free)(CUdeviceptr, size_t);
};

static bool drv_vmm(DrvVmm* d) {
    cudaDriverEntryPointQueryResult q;
    const char* names[8] = {"cuMemGetAllocationGranularity", "cuMemAddressReserve", "cuMemCreate", "cuMemMap",
                            "cuMemSetAccess", "cuMemUnmap", "cuMemRelease", "cuMemAddressFree"};
    void** slots[8] = {(void**)&d->granularity, (void**)&d->reserve, (void**)&d->create, (void**)&d->map,
                       (void**)&d->access, (void**)&d->unmap, (void**)&d->release, (void**)&d->addr_free};
    for (int i = 0; i < 8; i++)
        if (cudaGetDriverEntryPoint(names[i], slots[i], cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return false;
    return true;
}

// Device buffer for the benchmark: 0 = cudaMalloc, 1 = VMM (cuMemCreate +
// cuMemMap at the recommended granularity), 2 = stream-ordered pool.
static int rr_alloc(int kind, uint64_t bytes, void** p, uint64_t* gran, CUmemGenericAllocationHandle* h) {
    *gran = 0;
    if (kind == 1) {
        DrvVmm D;
        if (!drv_vmm(&D)) {
            set_error("driver VMM entry points unavailable");
            return GX_EINTERNAL;
        }
        int dev = 0;
        GX_CUDA(cudaGetDevice(&dev));
        CUmemAllocationProp prop = {};
        prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
        prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        prop.location.id = dev;
        size_t g = 0;
        if (D.granularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS) {
            set_error("cuMemGetAllocationGranularity failed");
            return GX_EINTERNAL;
        }
        *gran = g;
        bytes = (bytes + g - 1) / g * g;
        CUdeviceptr va = 0;
        if (D.reserve(&va, bytes, g, 0, 0) != CUDA_SUCCESS || D.create(h, bytes, &prop, 0) != CUDA_SUCCESS ||
            D.map(va, bytes, 0, *h, 0) != CUDA_SUCCESS) {
            set_error("VMM allocation failed");
            return GX_EINTERNAL;
        }
        CUmemAccessDesc acc = {};
        acc.location = prop.location;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        if (D.access(va, bytes, &acc, 1) != CUDA_SUCCESS) {
            set_error("cuMemSetAccess failed");
            return GX_EINTERNAL;
        }
        *p = (void*)va;
        return GX_OK;
    }
    if (kind == 2) {
        GX_CUDA(cudaMallocAsync(p, bytes, 0));
        GX_CUDA(cudaStreamSynchronize(0));
        return GX_OK;
    }
    GX_CUDA(cudaMalloc(p, bytes));
    return GX_OK;
}

static void rr_free(int kind, void* p, uint64_t bytes, uint64_t gran, CUmemGenericAllocationHandle h) {
    if (kind == 1) {
        DrvVmm D;
        if (!drv_vmm(&D)) return;
        bytes = (bytes + gran - 1) / gran * gran;
        D.unmap((CUdeviceptr)p, bytes);
        D.release(h);
        D.addr_free((CUdeviceptr)p, bytes);
    } else if (kind == 2) {
        cudaFreeAsync(p, 0);
        cudaStreamSynchronize(0);
    } else {
        cudaFree(p);
    }
}

extern "C" int gx_random_access_bench(uint64_t buffer_bytes, int32_t granularity, uint64_t reads,
                                      int32_t with_cas, int32_t repeats, double* ms_best,
                                      double* gbs_best) {
    return gx_random_access_bench_alloc(buffer_bytes, granularity, reads, with_cas, repeats, 0, ms_best,
                                        gbs_best, nullptr);
}

extern "C" int gx_random_access_bench_alloc(uint64_t buffer_bytes, int32_t granularity, uint64_t reads,
                                            int32_t with_cas, int32_t repeats, int32_t alloc_kind,
                                            double* ms_best, double* gbs_best, uint64_t* alloc_granularity) {
    rr_kernel_t k = with_cas ? pick_rr<true>(granularity) : pick_rr<false>(granularity);
    if (!k || buffer_bytes < (uint64_t)granularity || reads == 0 || repeats < 1) {
        set_error("random_access_bench: granularity must be 16/32/64/128 and sizes positive");
        return GX_EINPUT;
    }
    void* buf = nullptr;
    unsigned long long* sink = nullptr;
    uint64_t gran = 0;
    CUmemGenericAllocationHandle vh = 0;
    int rc = rr_alloc(alloc_kind, buffer_bytes, &buf, &gran, &vh);
    if (rc) return rc;
    if (alloc_granularity) *alloc_granularity = gran;
    GX_CUDA(cudaMalloc(&sink, 8));
    GX_CUDA(cudaMemset(buf, 0, buffer_bytes));
    const uint64_t segments = buffer_bytes / granularity;
    const int grid = sm_count() * 8;
    cudaEvent_t a, b;
    GX_CUDA(cudaEventCreate(&a));
    GX_CUDA(cudaEventCreate(&b));
    float best = 1e30f;
    for (int r = 0; r < repeats + 1; r++) {  // first launch is warm-up
        GX_CUDA(cudaEventRecord(a));
        k<<<grid, 256>>>((const uint4*)buf, segments, reads, 0x1234567ull * (r + 1), sink);
        GX_LAUNCHED();
        GX_CUDA(cudaEventRecord(b));
        GX_CUDA(cudaEventSynchronize(b));
        float ms = 0;
        GX_CUDA(cudaEventElapsedTime(&ms, a, b));
        if (r > 0 && ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    rr_free(alloc_kind, buf, buffer_bytes, gran, vh);
    cudaFree(sink);
    *ms_best = best;
    *gbs_best = (double)reads * granularity / (best * 1e-3) / 1e9;
    return GX_OK;
}
