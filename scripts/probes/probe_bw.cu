// Per-SM streaming-bandwidth probe: each CTA streams `per_cta` bytes from HBM into a
// shared-memory ring with cp.async.bulk (1D, contiguous) or TMA 2D boxes (128 rows x
// 128 B, row stride `stride`), `stages` in flight. Prints GB/s per SM and total.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c));
}
__device__ __forceinline__ void expect_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mwait(unsigned long long* b, unsigned ph) {
    asm volatile("{\n.reg .pred P;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W_%=;\n}" ::"r"(
                     smem_u32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, unsigned long long* bar, int c0, int c1) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                     smem_u32(dst)), "l"((unsigned long long)m), "r"(smem_u32(bar)), "r"(c0), "r"(c1) : "memory");
}

__global__ void stream_kernel(const char* src, size_t per_cta, int stage_bytes, int stages, int mode,
                              const __grid_constant__ CUtensorMap map, int kb_per_cta, int* sink, int nsplit) {
    extern __shared__ __align__(1024) unsigned char sm[];
    unsigned long long* bar = (unsigned long long*)(sm + stages * stage_bytes);
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) mbar_init(&bar[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (mode == 3) {
        // two issuing warps: warp w owns stages s with s % 2 == w
        const int w = threadIdx.x >> 5;
        if ((threadIdx.x & 31) != 0 || w > 1) return;
        const char* base = src + (size_t)blockIdx.x * per_cta;
        const int n = (int)(per_cta / stage_bytes);
        int acc = 0;
        for (int i = w; i < n + stages; i += 2) {
            if (i >= stages) {
                const int j = i - stages, s = j % stages;
                mwait(&bar[s], (j / stages) & 1);
                acc += sm[s * stage_bytes];
            }
            if (i < n) {
                const int s = i % stages;
                expect_tx(&bar[s], stage_bytes);
                bulk(sm + s * stage_bytes, base + (size_t)i * stage_bytes, stage_bytes, &bar[s]);
            }
        }
        if (acc == 12345) sink[0] = acc;
        return;
    }
    if (threadIdx.x != 0) return;
    const char* base = src + (size_t)blockIdx.x * per_cta;
    const int n = mode == 0 ? (int)(per_cta / stage_bytes) : kb_per_cta;
    int acc = 0;
    for (int i = 0; i < n + stages; ++i) {
        if (i >= stages) {
            const int j = i - stages, s = j % stages;
            mwait(&bar[s], (j / stages) & 1);
            acc += sm[s * stage_bytes];
        }
        if (i < n) {
            const int s = i % stages;
            expect_tx(&bar[s], stage_bytes);
            if (mode == 0) bulk(sm + s * stage_bytes, base + (size_t)i * stage_bytes, stage_bytes, &bar[s]);
            else if (mode == 2) {
                const int piece = stage_bytes / nsplit;
                for (int p = 0; p < nsplit; ++p)
                    bulk(sm + s * stage_bytes + p * piece, base + (size_t)i * stage_bytes + p * piece, piece, &bar[s]);
            }
            else {
                // 16 KB = one 64-col x 128-row box; stage_bytes/16K boxes along rows
                for (int b = 0; b < stage_bytes / 16384; ++b)
                    tma2d(sm + s * stage_bytes + b * 16384, &map, &bar[s], i * 64, blockIdx.x * 128 * (stage_bytes / 16384) + b * 128);
            }
        }
    }
    if (acc == 12345) sink[0] = acc;
}

int main() {
    size_t total = (size_t)2 << 30;
    char* d;
    cudaMalloc(&d, total);
    cudaMemset(d, 1, total);
    int* sink;
    cudaMalloc(&sink, 4);
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    // TMA map: weight-like [rows][K] bf16, K = 8960
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    const int K = 8960;
    const unsigned long long rows = total / (K * 2);
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)K, rows};
    cuuint64_t str[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    struct Case { int mode, sb, st, ctas, nsplit; };
    std::vector<Case> cases = {
        {0, 16384, 8, 1, 1}, {2, 16384, 8, 1, 4}, {2, 65536, 2, 1, 4}, {2, 65536, 2, 1, 16}, {3, 16384, 8, 1, 1},
        {0, 8192, 16, 1, 1}, {0, 131072, 1, 1, 1}, {2, 131072, 1, 1, 8}, {0, 16384, 8, 16, 1}, {2, 65536, 3, 1, 1},
        {0, 65536, 3, 1, 1}, {0, 32768, 6, 1, 1}};
    for (auto c : cases) {
        size_t per = (size_t)4 << 20;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            stream_kernel<<<c.ctas, 64, c.sb * c.st + 256>>>(d, per, c.sb, c.st, c.mode, map, 140, sink, c.nsplit);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        double gb = (double)per * c.ctas / 1e9;
        printf("{\"mode\": %d, \"stage_KB\": %d, \"stages\": %d, \"nsplit\": %d, \"ctas\": %d, \"GBps_per_sm\": %.1f}\n", c.mode,
               c.sb / 1024, c.st, c.nsplit, c.ctas, gb / (ms * 1e-3) / c.ctas);
    }
    cudaError_t e = cudaGetLastError();
    printf("err %s\n", cudaGetErrorString(e));
}
