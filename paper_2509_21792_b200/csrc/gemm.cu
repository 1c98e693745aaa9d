// tcgen05 + TMA GEMM for sm_100a:  P[s][t][o] = sum_{k in split s} X[t][k] * W[o][k]
//
// Replaces the reference's scalar i-k-j nn::matmul (include/sgrpo/nn.hpp:15-29) for every
// projection of the decode forward (tinylm.hpp:325-327 q/k/v, :396 wo, :400 w1, :402 w2,
// :458 lm_head, :528 w_fuse). Weights live on the device K-major ([out][in], bf16), so
// y = x.W of the reference becomes a "TN" GEMM with the weight as the UMMA A operand
// (M = 128 output features per tile) and the token rows as the B operand (N = BN tokens).
// This swap-AB mapping keeps the tensor core busy at decode batch sizes (1..256 rows),
// where the kernel streams weight tiles at HBM rate.
//
// Batch invariance (SURVEY.md §7 hard part 1): the K split (grid.y) is a function of the
// weight shape only, each output element accumulates its K range in the same order for
// every BN, and partial sums are reduced in split order by the epilogue kernels
// (rowops.cu). A row's result therefore never depends on how many rows share the launch.
#include <cudaTypedefs.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#include "common.cuh"
#include "gemm.h"

namespace sgb {

namespace {

constexpr int kBK = 64;          // 64 bf16 = 128 B = one swizzle row
constexpr int kBM = 128;         // output features per tile (UMMA M)
constexpr int kABytes = kBM * kBK * 2;

template <int BN>
struct GemmCfg {
    static constexpr int kBBytes = BN * kBK * 2;
    static constexpr int kStage = kABytes + kBBytes;
    static constexpr int kStages = (200 * 1024) / kStage > 8 ? 8 : (200 * 1024) / kStage;
    static constexpr int kTmemCols = BN < 32 ? 32 : BN;
    static constexpr int kSmem = kStages * kStage + 1024 /*align*/ + 256 /*barriers*/;
};

template <int BN>
__global__ void __launch_bounds__(128, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap mapW, const __grid_constant__ CUtensorMap mapX,
                        float* __restrict__ out, int M, int N, int kb_per_split, int kb_total) {
    using Cfg = GemmCfg<BN>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::kStages * Cfg::kStage);
    uint64_t* empty = full + Cfg::kStages;
    uint64_t* done = empty + Cfg::kStages;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int m0 = blockIdx.x * BN;
    const int n0 = blockIdx.y * kBM;
    const int split = blockIdx.z;
    const int kb0 = split * kb_per_split;
    const int nkb = min(kb_per_split, kb_total - kb0);

    if (warp == 0 && lane == 0) {
        tma_prefetch(&mapW);
        tma_prefetch(&mapX);
        for (int s = 0; s < Cfg::kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_barrier_init();
    }
    if (warp == 1) tmem_alloc<Cfg::kTmemCols>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // TMA producer: weights are streamed once (evict-first), activations stay in L2.
        const uint64_t pol_w = policy_evict_first();
        for (int i = 0; i < nkb; ++i) {
            const int s = i % Cfg::kStages;
            if (i >= Cfg::kStages) mbar_wait(&empty[s], ((i / Cfg::kStages) & 1) ^ 1);
            uint8_t* a = smem + s * Cfg::kStage;
            mbar_arrive_expect_tx(&full[s], Cfg::kStage);
            tma_load_2d_hint(a, &mapW, &full[s], (kb0 + i) * kBK, n0, pol_w);
            tma_load_2d(a + kABytes, &mapX, &full[s], (kb0 + i) * kBK, m0);
        }
    } else if (warp == 1 && lane == 0) {
        // MMA issuer: one thread drives the tensor core; accumulator lives in TMEM.
        constexpr uint32_t idesc = idesc_bf16_m128(BN);
        for (int i = 0; i < nkb; ++i) {
            const int s = i % Cfg::kStages;
            mbar_wait(&full[s], (i / Cfg::kStages) & 1);
            tc_fence_after();
            const uint32_t a = smem_u32(smem + s * Cfg::kStage);
            const uint64_t adesc = sw128_desc(a), bdesc = sw128_desc(a + kABytes);
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
                umma_bf16(tmem, adesc + 2 * k, bdesc + 2 * k, idesc, (i | k) != 0);
            umma_commit(&empty[s]);
        }
        umma_commit(done);
    }
    __syncwarp();
    mbar_wait(done, 0);
    tc_fence_after();

    // Epilogue: warp w owns TMEM lanes [32w, 32w+32) = output features n0+32w+lane; the
    // columns are token rows. Stores are coalesced along the feature dimension.
    const int o = n0 + 32 * warp + lane;
    float* dst = out + static_cast<size_t>(split) * M * N;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 16) {
        if (m0 + c0 >= M) break;
        float v[16];
        tmem_ld16(tmem + (static_cast<uint32_t>(32 * warp) << 16) + c0, v);
        if (o < N) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int t = m0 + c0 + j;
                if (t < M) dst[static_cast<size_t>(t) * N + o] = v[j];
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc<Cfg::kTmemCols>(tmem);
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p)
            throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

template <int BN>
void launch_bn(const CUtensorMap& w, const CUtensorMap& x, float* out, int M, int N, int S, int kbps, int kbt,
               cudaStream_t st) {
    using Cfg = GemmCfg<BN>;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(gemm_bf16_tn_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem);
        attr = true;
    }
    dim3 grid((M + BN - 1) / BN, (N + kBM - 1) / kBM, S);
    gemm_bf16_tn_kernel<BN><<<grid, 128, Cfg::kSmem, st>>>(w, x, out, M, N, kbps, kbt);
}

}  // namespace

CUtensorMap make_kmajor_map(const void* ptr, int rows, int K, int box_rows) {
    if (K % 8) throw std::invalid_argument("GEMM K must be a multiple of 8");
    CUtensorMap m;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(K) * 2};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                              estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return m;
}

int gemm_splits(int N, int K) {
    const int tiles_n = (N + kBM - 1) / kBM;
    const int kbt = (K + kBK - 1) / kBK;
    int want = (2 * 148 + tiles_n - 1) / tiles_n;  // ~2 CTAs per SM worth of tiles
    if (want > 16) want = 16;
    if (want > kbt / 2) want = kbt / 2;  // keep >= 2 k-blocks per split
    if (want < 1) want = 1;
    const int kbps = (kbt + want - 1) / want;
    return (kbt + kbps - 1) / kbps;
}

int gemm_bn_for(int M) {
    if (M <= 16) return 16;
    if (M <= 32) return 32;
    if (M <= 64) return 64;
    if (M <= 128) return 128;
    return 256;
}

void gemm_launch(const GemmWeight& w, const GemmAct& x, float* partials, int M, cudaStream_t st) {
    if (M <= 0) return;
    const int kbt = (w.K + kBK - 1) / kBK;
    const int kbps = (kbt + w.splits - 1) / w.splits;
    const int S = (kbt + kbps - 1) / kbps;
    const int bn = gemm_bn_for(M);
    const CUtensorMap& xm = x.map_for_bn(bn);
    switch (bn) {
        case 16: launch_bn<16>(w.map, xm, partials, M, w.N, S, kbps, kbt, st); break;
        case 32: launch_bn<32>(w.map, xm, partials, M, w.N, S, kbps, kbt, st); break;
        case 64: launch_bn<64>(w.map, xm, partials, M, w.N, S, kbps, kbt, st); break;
        case 128: launch_bn<128>(w.map, xm, partials, M, w.N, S, kbps, kbt, st); break;
        default: launch_bn<256>(w.map, xm, partials, M, w.N, S, kbps, kbt, st); break;
    }
}

void GemmWeight::init(const __nv_bfloat16* p, int n, int k) {
    ptr = p;
    N = n;
    K = k;
    splits = gemm_splits(n, k);
    map = make_kmajor_map(p, n, k, kBM);
}

void GemmAct::init(const __nv_bfloat16* p, int rows, int k) {
    ptr = p;
    cap_rows = rows;
    K = k;
    const int bns[5] = {16, 32, 64, 128, 256};
    for (int i = 0; i < 5; ++i) maps[i] = make_kmajor_map(p, rows, k, bns[i]);
}

const CUtensorMap& GemmAct::map_for_bn(int bn) const {
    switch (bn) {
        case 16: return maps[0];
        case 32: return maps[1];
        case 64: return maps[2];
        case 128: return maps[3];
        default: return maps[4];
    }
}

}  // namespace sgb
