// Test-only entry points (libsgrpo_b200_dev.so, declared in include/sgrpo_b200_dev.h): kernel
// self-tests on host-supplied operands and microbenchmarks. They link the same kernels as the
// product library but are not part of the drop-in boundary; tests and scripts/ load them.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "sgrpo_b200_dev.h"
#include "../csrc/engine.h"
#include "../csrc/gemm.h"
#include "../csrc/kernels.h"
#include "../csrc/util.h"

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return sgb::SGB_OK;
    } catch (const sgb::CudaError& e) {
        g_err = e.what();
        return sgb::SGB_ECUDA;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return sgb::SGB_EINVAL;
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return sgb::SGB_ERANGE;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return sgb::SGB_EDOMAIN;
    } catch (const std::exception& e) {
        g_err = e.what();
        return sgb::SGB_ERUNTIME;
    }
}
}  // namespace

extern "C" {

const char* sgb_dev_last_error(void) { return g_err.c_str(); }

int sgb_debug_group_advantages(const int* tokens, const int* lens, const int* prompt_lens, int n_groups, int g,
                               int stride, const long long* answers, double eps_var, double* rewards,
                               double* advantages, int* valid) {
    return guarded([&] {
        if (n_groups <= 0 || g < 2) throw std::invalid_argument("standardize_advantages: need G >= 2");
        const int n = n_groups * g;
        for (int s = 0; s < n; ++s)
            if (lens[s] < prompt_lens[s] || lens[s] > stride || prompt_lens[s] < 0)
                throw std::invalid_argument("group_advantages: bad sequence lengths");
        int *dt = nullptr, *dl = nullptr, *dp = nullptr, *dv = nullptr;
        long long* da = nullptr;
        double* db = nullptr;
        SGB_CUDA(cudaMalloc(&dt, sizeof(int) * static_cast<size_t>(n) * stride));
        SGB_CUDA(cudaMalloc(&dl, sizeof(int) * n));
        SGB_CUDA(cudaMalloc(&dp, sizeof(int) * n));
        SGB_CUDA(cudaMalloc(&dv, sizeof(int) * n_groups));
        SGB_CUDA(cudaMalloc(&da, sizeof(long long) * n_groups));
        SGB_CUDA(cudaMalloc(&db, sizeof(double) * 2 * n));
        SGB_CUDA(cudaMemcpy(dt, tokens, sizeof(int) * static_cast<size_t>(n) * stride, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dl, lens, sizeof(int) * n, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dp, prompt_lens, sizeof(int) * n, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(da, answers, sizeof(long long) * n_groups, cudaMemcpyHostToDevice));
        sgb::launch_group_advantages(n_groups, g, dt, stride, dl, dp, da, eps_var, db, db + n, dv, 0);
        SGB_CUDA(cudaDeviceSynchronize());
        SGB_CUDA(cudaMemcpy(rewards, db, sizeof(double) * n, cudaMemcpyDeviceToHost));
        SGB_CUDA(cudaMemcpy(advantages, db + n, sizeof(double) * n, cudaMemcpyDeviceToHost));
        SGB_CUDA(cudaMemcpy(valid, dv, sizeof(int) * n_groups, cudaMemcpyDeviceToHost));
        void* ptrs[] = {dt, dl, dp, dv, da, db};
        for (void* p : ptrs) cudaFree(p);
    });
}

// GEMM microbenchmark: device-resident random bf16 operands, fused fp32 epilogue,
// average device ms over `iters` launches (CUDA events on the launching stream).
int sgb_bench_gemm(int M, int N, int K, int splits, int iters, double* ms_out) {
    return guarded([&] {
        const int cap = ((M + 255) / 256) * 256;
        // Weights rotate over enough copies to exceed the 126 MB L2, so every launch streams
        // its weights from HBM as in the rollout (28 layers x 74 MB at the c2 shape).
        const size_t wbytes = static_cast<size_t>(N) * K * 2;
        const int ncopy = static_cast<int>(std::max<size_t>(1, (320u << 20) / wbytes + 1));
        std::vector<__nv_bfloat16> hw(static_cast<size_t>(N) * K), hx(static_cast<size_t>(cap) * K);
        uint64_t st = 12345;
        auto rnd = [&]() {
            st = st * 6364136223846793005ULL + 1442695040888963407ULL;
            return static_cast<float>((st >> 40) & 0xFFFF) / 65536.0f - 0.5f;
        };
        for (auto& v : hw) v = __float2bfloat16(0.05f * rnd());
        for (auto& v : hx) v = __float2bfloat16(rnd());
        __nv_bfloat16 *dw = nullptr, *dx = nullptr;
        float* dp = nullptr;
        SGB_CUDA(cudaMalloc(&dw, wbytes * ncopy));
        SGB_CUDA(cudaMalloc(&dx, hx.size() * 2));
        for (int c = 0; c < ncopy; ++c)
            SGB_CUDA(cudaMemcpy(reinterpret_cast<char*>(dw) + c * wbytes, hw.data(), wbytes, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dx, hx.data(), hx.size() * 2, cudaMemcpyHostToDevice));
        std::vector<sgb::GemmWeight> gw(ncopy);
        for (int c = 0; c < ncopy; ++c)
            gw[c].init(reinterpret_cast<const __nv_bfloat16*>(reinterpret_cast<const char*>(dw) + c * wbytes), N, K);
        sgb::GemmAct ga;
        ga.init(dx, cap, K);
        sgb::GemmWorkspace ws;
        ws.cap_floats = sgb::gemm_ws_floats(M, N, K);
        ws.ctr_cap = 1 << 16;
        SGB_CUDA(cudaMalloc(&ws.buf, ws.cap_floats * 4));
        SGB_CUDA(cudaMalloc(&ws.ctr, ws.ctr_cap * sizeof(int)));
        SGB_CUDA(cudaMemset(ws.ctr, 0, ws.ctr_cap * sizeof(int)));
        // splits < 0: kEpiPartials (raw chunk sums, one unit per (tile, chunk))
        const size_t out_floats = static_cast<size_t>(M) * N * (splits < 0 ? sgb::gemm_chunks(N, K) : 1);
        SGB_CUDA(cudaMalloc(&dp, out_floats * 4));
        sgb::GemmEpi epi;
        epi.kind = splits < 0 ? sgb::kEpiPartials : sgb::kEpiF32;
        epi.f32 = dp;
        epi.ld = N;
        if (splits < 0) splits = 0;
        cudaEvent_t a, b;
        SGB_CUDA(cudaEventCreate(&a));
        SGB_CUDA(cudaEventCreate(&b));
        for (int i = 0; i < 3; ++i) sgb::gemm_run(gw[i % ncopy], ga, M, epi, ws, 0, splits);
        SGB_CUDA(cudaEventRecord(a, 0));
        for (int i = 0; i < iters; ++i) sgb::gemm_run(gw[(i + 3) % ncopy], ga, M, epi, ws, 0, splits);
        SGB_CUDA(cudaEventRecord(b, 0));
        SGB_CUDA(cudaEventSynchronize(b));
        SGB_KCHECK();
        float ms = 0.f;
        SGB_CUDA(cudaEventElapsedTime(&ms, a, b));
        *ms_out = ms / iters;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaFree(dw);
        cudaFree(dx);
        cudaFree(dp);
        cudaFree(ws.buf);
        cudaFree(ws.ctr);
    });
}

// Attention self-test: row r attends to n_keys[r] keys stored consecutively (rows
// concatenated) in K/V [sum n_keys][H*dh]; the LAST key of every row is addressed through
// the tree-path (chain) slot list, the rest as the contiguous cached prefix. out [B][H*dh].
int sgb_debug_attention(int B, const int* n_keys, int H, int dh, const float* q, const float* k, const float* v,
                        float* out) {
    return guarded([&] {
        if (B <= 0 || H <= 0 || dh <= 0) throw std::invalid_argument("debug_attention: bad shape");
        const int d = H * dh;
        std::vector<long long> base(B), chain(static_cast<size_t>(B) * sgb::kMaxChain, 0);
        std::vector<int> cl(B), chl(B, 1);
        long long tot = 0;
        int maxk = 1;
        double keys = 0;
        for (int b = 0; b < B; ++b) {
            if (n_keys[b] < 1) throw std::invalid_argument("debug_attention: rows need >= 1 key");
            base[b] = tot;
            cl[b] = n_keys[b] - 1;
            chain[static_cast<size_t>(b) * sgb::kMaxChain] = tot + n_keys[b] - 1;
            tot += n_keys[b];
            maxk = std::max(maxk, n_keys[b]);
            keys += n_keys[b];
        }
        std::vector<__nv_bfloat16> hk(tot * d), hv(tot * d);
        for (size_t i = 0; i < hk.size(); ++i) {
            hk[i] = __float2bfloat16(k[i]);
            hv[i] = __float2bfloat16(v[i]);
        }
        __nv_bfloat16 *K = nullptr, *V = nullptr, *o = nullptr;
        float *dq = nullptr, *pacc = nullptr, *pml = nullptr;
        long long *dbase = nullptr, *dchain = nullptr;
        int *dcl = nullptr, *dchl = nullptr;
        const int ns = sgb::attn_splits_for(maxk);
        SGB_CUDA(cudaMalloc(&K, hk.size() * 2));
        SGB_CUDA(cudaMalloc(&V, hv.size() * 2));
        SGB_CUDA(cudaMalloc(&o, static_cast<size_t>(B) * d * 2));
        SGB_CUDA(cudaMalloc(&dq, static_cast<size_t>(B) * d * 4));
        SGB_CUDA(cudaMalloc(&pacc, static_cast<size_t>(B) * d * ns * 4));
        SGB_CUDA(cudaMalloc(&pml, static_cast<size_t>(B) * H * ns * 2 * 4));
        SGB_CUDA(cudaMalloc(&dbase, B * 8));
        SGB_CUDA(cudaMalloc(&dchain, chain.size() * 8));
        SGB_CUDA(cudaMalloc(&dcl, B * 4));
        SGB_CUDA(cudaMalloc(&dchl, B * 4));
        SGB_CUDA(cudaMemcpy(K, hk.data(), hk.size() * 2, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(V, hv.data(), hv.size() * 2, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dq, q, static_cast<size_t>(B) * d * 4, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dbase, base.data(), B * 8, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dchain, chain.data(), chain.size() * 8, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dcl, cl.data(), B * 4, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dchl, chl.data(), B * 4, cudaMemcpyHostToDevice));
        sgb::AttnRowsDev ar{dbase, dcl, dchl, dchain};
        sgb::AttnScratch sc{pacc, pml, nullptr, static_cast<long long>(B) * H};
        SGB_CUDA(cudaMalloc(&sc.row_ctr, sc.ctr_cap * 4));
        SGB_CUDA(cudaMemset(sc.row_ctr, 0, sc.ctr_cap * 4));
        sgb::launch_attention(dq, K, V, tot, ar, B, H, d, maxk, keys, sc, o, 0);
        SGB_CUDA(cudaDeviceSynchronize());
        std::vector<__nv_bfloat16> ho(static_cast<size_t>(B) * d);
        SGB_CUDA(cudaMemcpy(ho.data(), o, ho.size() * 2, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < ho.size(); ++i) out[i] = __bfloat162float(ho[i]);
        void* ptrs[] = {K, V, o, dq, pacc, pml, dbase, dchain, dcl, dchl, sc.row_ctr};
        for (void* p : ptrs) cudaFree(p);
    });
}

namespace {
// Device state of a tree-attention case: n_groups sequences, each with ctx_len committed keys
// and a tree of rows (level order, parent within the group) -- the verify rows of one step.
struct TreeAttnCase {
    int M = 0, H = 0, d = 0, max_vlen = 1, n_tiles = 0, qw = 1;
    long long items = 0, n_slots = 0;
    double keys = 0;
    std::vector<void*> ptrs;
    __nv_bfloat16 *K = nullptr, *V = nullptr, *o1 = nullptr, *o2 = nullptr;
    float* q = nullptr;
    sgb::AttnRowsDev ar{};
    sgb::AttnScratch sc{};
    sgb::AttnTileDev* tiles = nullptr;
    std::vector<sgb::TreeGroupDev> tg;
    sgb::TreeGroupDev* dtg = nullptr;
    sgb::TreeTileDev* dtt = nullptr;
    int tw = 1, n_ttiles = 0, max_nodes = 1;
    CUtensorMap kmap, vmap;

    void* dev(size_t bytes) {
        void* p = nullptr;
        SGB_CUDA(cudaMalloc(&p, std::max<size_t>(bytes, 16)));
        ptrs.push_back(p);
        return p;
    }
    TreeAttnCase(int n_groups, const int* ctx_len, const int* n_rows, const int* parent, int H_, int dh,
                 const float* hq, const float* kctx, const float* vctx, const float* knode, const float* vnode)
        : H(H_), d(H_ * dh) {
        if (n_groups <= 0 || H <= 0 || dh <= 0) throw std::invalid_argument("tree_attention: bad shape");
        long long n_ctx = 0;
        for (int g = 0; g < n_groups; ++g) {
            if (ctx_len[g] < 0 || n_rows[g] < 1) throw std::invalid_argument("tree_attention: bad group");
            n_ctx += ctx_len[g];
            M += n_rows[g];
        }
        // KV store: committed keys of every group, then one node slot per row
        const long long slots = n_ctx + M;
        n_slots = slots;
        std::vector<long long> base(M), chain(static_cast<size_t>(M) * sgb::kMaxChain, 0);
        std::vector<int> cl(M), chl(M);
        std::vector<sgb::AttnTileDev> ht;
        std::vector<std::array<int, 4>> groups;
        long long cbase = 0;
        int row = 0;
        for (int g = 0; g < n_groups; ++g) {
            const int r0 = row;
            std::vector<int> depth(n_rows[g]);
            int gmax = 1;
            for (int i = 0; i < n_rows[g]; ++i, ++row) {
                const int p = parent[row];
                if (i == 0 ? p != -1 : (p < 0 || p >= i)) throw std::invalid_argument("tree_attention: bad parent");
                depth[i] = i == 0 ? 0 : depth[p] + 1;
                if (depth[i] + 1 > sgb::kMaxChain) throw std::invalid_argument("tree_attention: tree too deep");
                base[row] = cbase;
                cl[row] = ctx_len[g];
                chl[row] = depth[i] + 1;
                for (int a = i; a >= 0; a = a == 0 ? -1 : parent[r0 + a])
                    chain[static_cast<size_t>(row) * sgb::kMaxChain + depth[a]] = n_ctx + r0 + a;
                gmax = std::max(gmax, ctx_len[g] + depth[i] + 1);
                keys += ctx_len[g] + depth[i] + 1;
            }
            max_vlen = std::max(max_vlen, gmax);
            groups.push_back({r0, n_rows[g], ctx_len[g], gmax});
            cbase += ctx_len[g];
        }
        qw = sgb::attn_tile_qw(groups);
        items = sgb::build_attn_tiles(groups, ht, qw, true);
        n_tiles = static_cast<int>(ht.size());
        const int ns = sgb::attn_splits_for(max_vlen);
        K = static_cast<__nv_bfloat16*>(dev(static_cast<size_t>(slots) * d * 2));
        V = static_cast<__nv_bfloat16*>(dev(static_cast<size_t>(slots) * d * 2));
        o1 = static_cast<__nv_bfloat16*>(dev(static_cast<size_t>(M) * d * 2));
        o2 = static_cast<__nv_bfloat16*>(dev(static_cast<size_t>(M) * d * 2));
        q = static_cast<float*>(dev(static_cast<size_t>(M) * d * 4));
        if (hq) {
            std::vector<__nv_bfloat16> hk(static_cast<size_t>(slots) * d), hv(hk.size());
            for (size_t i = 0; i < static_cast<size_t>(n_ctx) * d; ++i) {
                hk[i] = __float2bfloat16(kctx[i]);
                hv[i] = __float2bfloat16(vctx[i]);
            }
            for (size_t i = 0; i < static_cast<size_t>(M) * d; ++i) {
                hk[n_ctx * d + i] = __float2bfloat16(knode[i]);
                hv[n_ctx * d + i] = __float2bfloat16(vnode[i]);
            }
            SGB_CUDA(cudaMemcpy(K, hk.data(), hk.size() * 2, cudaMemcpyHostToDevice));
            SGB_CUDA(cudaMemcpy(V, hv.data(), hv.size() * 2, cudaMemcpyHostToDevice));
            SGB_CUDA(cudaMemcpy(q, hq, static_cast<size_t>(M) * d * 4, cudaMemcpyHostToDevice));
        } else {  // timing only: constant data
            SGB_CUDA(cudaMemset(K, 0x3c, static_cast<size_t>(slots) * d * 2));
            SGB_CUDA(cudaMemset(V, 0x3c, static_cast<size_t>(slots) * d * 2));
            SGB_CUDA(cudaMemset(q, 0, static_cast<size_t>(M) * d * 4));
        }
        auto* pacc = static_cast<float*>(dev(static_cast<size_t>(M) * d * ns * 4));
        auto* pml = static_cast<float*>(dev(static_cast<size_t>(M) * H * ns * 2 * 4));
        auto* dbase = static_cast<long long*>(dev(M * 8));
        auto* dchain = static_cast<long long*>(dev(chain.size() * 8));
        auto* dcl = static_cast<int*>(dev(M * 4));
        auto* dchl = static_cast<int*>(dev(M * 4));
        tiles = static_cast<sgb::AttnTileDev*>(dev(ht.size() * sizeof(sgb::AttnTileDev)));
        // attention_tree.cu: one group per sequence (node rows = its tree rows' own slots)
        {
            long long cb = 0;
            int r = 0, mx = 1;
            for (int g = 0; g < n_groups; ++g) {
                tg.push_back(sgb::TreeGroupDev{r, n_rows[g], ctx_len[g], n_rows[g], n_ctx + r, cb, cb, 0, 0});
                max_nodes = std::max(max_nodes, n_rows[g]);
                mx = std::max(mx, n_rows[g]);
                cb += ctx_len[g];
                r += n_rows[g];
            }
            tw = sgb::tree_attn_warps(mx, n_groups, H, dh, max_nodes);
            std::vector<sgb::TreeTileDev> tt;
            sgb::build_tree_tiles(tg, tw, tt);
            n_ttiles = static_cast<int>(tt.size());
            dtg = static_cast<sgb::TreeGroupDev*>(dev(tg.size() * sizeof(sgb::TreeGroupDev)));
            dtt = static_cast<sgb::TreeTileDev*>(dev(tt.size() * sizeof(sgb::TreeTileDev)));
            SGB_CUDA(cudaMemcpy(dtg, tg.data(), tg.size() * sizeof(sgb::TreeGroupDev), cudaMemcpyHostToDevice));
            SGB_CUDA(cudaMemcpy(dtt, tt.data(), tt.size() * sizeof(sgb::TreeTileDev), cudaMemcpyHostToDevice));
            kmap = sgb::make_kmajor_map(K, static_cast<int>(slots), d, 16);
            vmap = sgb::make_kmajor_map(V, static_cast<int>(slots), d, 16);
        }
        sc = sgb::AttnScratch{pacc, pml, nullptr, static_cast<long long>(M) * H};  // >= rows x head groups
        sc.row_ctr = static_cast<int*>(dev(sc.ctr_cap * 4));
        SGB_CUDA(cudaMemset(sc.row_ctr, 0, sc.ctr_cap * 4));
        SGB_CUDA(cudaMemcpy(dbase, base.data(), M * 8, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dchain, chain.data(), chain.size() * 8, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dcl, cl.data(), M * 4, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dchl, chl.data(), M * 4, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(tiles, ht.data(), ht.size() * sizeof(sgb::AttnTileDev), cudaMemcpyHostToDevice));
        ar = sgb::AttnRowsDev{dbase, dcl, dchl, dchain};
    }
    ~TreeAttnCase() {
        for (void* p : ptrs) cudaFree(p);
    }
    void run_row() { sgb::launch_attention(q, K, V, n_slots, ar, M, H, d, max_vlen, keys, sc, o1, 0); }
    void run_tree() {
        sgb::launch_attention_tree(q, kmap, vmap, 0, K, V, ar, dtg, dtt, n_ttiles, tw, H, d, max_nodes, o2, 0);
    }
    void run_decode() {
        int mc = 0;
        for (const auto& g : tg) {
            if (g.nrows != 1) throw std::invalid_argument("decode attention: one row per group");
            mc = std::max(mc, g.ctx_len);
        }
        sgb::launch_attention_decode(q, kmap, vmap, 0, K, V, dtg, static_cast<int>(tg.size()), mc, H, d, o2, 0);
    }
    void run_group() { sgb::launch_attention_tiles(q, K, V, n_slots, ar, M, tiles, n_tiles, items, qw, H, d, max_vlen, sc, o2,
                                                    0); }
    void read(const __nv_bfloat16* o, float* out) const {
        std::vector<__nv_bfloat16> ho(static_cast<size_t>(M) * d);
        SGB_CUDA(cudaMemcpy(ho.data(), o, ho.size() * 2, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < ho.size(); ++i) out[i] = __bfloat162float(ho[i]);
    }
};
}  // namespace

int sgb_debug_tree_attention(int n_groups, const int* ctx_len, const int* n_rows, const int* parent, int H, int dh,
                             const float* q, const float* kctx, const float* vctx, const float* knode,
                             const float* vnode, float* out_row, float* out_group) {
    return guarded([&] {
        if (!q) throw std::invalid_argument("debug_tree_attention: null inputs");
        TreeAttnCase c(n_groups, ctx_len, n_rows, parent, H, dh, q, kctx, vctx, knode, vnode);
        c.run_row();
        c.run_group();
        SGB_CUDA(cudaDeviceSynchronize());
        c.read(c.o1, out_row);
        c.read(c.o2, out_group);
    });
}

int sgb_debug_tree_attention_tree(int n_groups, const int* ctx_len, const int* n_rows, const int* parent, int H, int dh,
                                  const float* q, const float* kctx, const float* vctx, const float* knode,
                                  const float* vnode, float* out_tree) {
    return guarded([&] {
        if (!q) throw std::invalid_argument("debug_tree_attention: null inputs");
        TreeAttnCase c(n_groups, ctx_len, n_rows, parent, H, dh, q, kctx, vctx, knode, vnode);
        c.run_tree();
        SGB_CUDA(cudaDeviceSynchronize());
        c.read(c.o2, out_tree);
    });
}

// attention_tree.cu's cluster decode kernel (AR steps: one row per group) on the same inputs
int sgb_debug_attention_decode(int n_groups, const int* ctx_len, int H, int dh, const float* q, const float* kctx,
                               const float* vctx, const float* knode, const float* vnode, float* out_row,
                               float* out_decode) {
    return guarded([&] {
        if (!q) throw std::invalid_argument("debug_attention_decode: null inputs");
        std::vector<int> nr(n_groups, 1), par(n_groups, -1);
        TreeAttnCase c(n_groups, ctx_len, nr.data(), par.data(), H, dh, q, kctx, vctx, knode, vnode);
        c.run_row();
        c.run_decode();
        SGB_CUDA(cudaDeviceSynchronize());
        c.read(c.o1, out_row);
        c.read(c.o2, out_decode);
    });
}

// AR attention microbenchmark: B rows with ctx committed keys each; device ms per launch of
// attention.cu (row path), the tree kernel and the cluster decode kernel
int sgb_bench_attention_decode(int B, int ctx, int H, int dh, int iters, double* ms_row, double* ms_tree,
                               double* ms_decode) {
    return guarded([&] {
        if (B <= 0 || iters <= 0) throw std::invalid_argument("bench_attention_decode: bad shape");
        std::vector<int> cl(B, ctx), nr(B, 1), par(B, -1);
        TreeAttnCase c(B, cl.data(), nr.data(), par.data(), H, dh, nullptr, nullptr, nullptr, nullptr, nullptr);
        cudaEvent_t a, b;
        SGB_CUDA(cudaEventCreate(&a));
        SGB_CUDA(cudaEventCreate(&b));
        auto time = [&](auto&& f) {
            for (int i = 0; i < 2; ++i) f();
            SGB_CUDA(cudaEventRecord(a, 0));
            for (int i = 0; i < iters; ++i) f();
            SGB_CUDA(cudaEventRecord(b, 0));
            SGB_CUDA(cudaEventSynchronize(b));
            float ms = 0.f;
            SGB_CUDA(cudaEventElapsedTime(&ms, a, b));
            return static_cast<double>(ms) / iters;
        };
        *ms_row = time([&] { c.run_row(); });
        *ms_tree = time([&] { c.run_tree(); });
        *ms_decode = time([&] { c.run_decode(); });
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    });
}

int sgb_bench_tree_attention_tree(int B, int N, int ctx, int H, int dh, int iters, double* ms_tree) {
    return guarded([&] {
        if (B <= 0 || N <= 0 || iters <= 0) throw std::invalid_argument("bench_tree_attention: bad shape");
        std::vector<int> cl(B, ctx), nr(B, N), par;
        for (int b = 0; b < B; ++b) {
            std::vector<int> dep(N, 0);
            for (int i = 0; i < N; ++i) {
                int p = i == 0 ? -1 : (i - 1) / 10;
                if (i) {
                    while (dep[p] + 1 >= sgb::kMaxChain) p = (p - 1) / 10;
                    dep[i] = dep[p] + 1;
                }
                par.push_back(p);
            }
        }
        TreeAttnCase c(B, cl.data(), nr.data(), par.data(), H, dh, nullptr, nullptr, nullptr, nullptr, nullptr);
        cudaEvent_t a, b;
        SGB_CUDA(cudaEventCreate(&a));
        SGB_CUDA(cudaEventCreate(&b));
        for (int i = 0; i < 2; ++i) c.run_tree();
        SGB_CUDA(cudaEventRecord(a, 0));
        for (int i = 0; i < iters; ++i) c.run_tree();
        SGB_CUDA(cudaEventRecord(b, 0));
        SGB_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        SGB_CUDA(cudaEventElapsedTime(&ms, a, b));
        *ms_tree = ms / iters;
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    });
}

// Tree-verify attention microbenchmark: B sequences with ctx committed keys each, an EAGLE-
// shaped tree of N rows per sequence (node i's parent (i-1)/k, depth <= kMaxChain-1); times
// the per-row kernel and the prefix-shared group kernel (CUDA events, default stream).
int sgb_bench_tree_attention(int B, int N, int ctx, int H, int dh, int iters, double* ms_row, double* ms_group) {
    return guarded([&] {
        if (B <= 0 || N <= 0 || iters <= 0) throw std::invalid_argument("bench_tree_attention: bad shape");
        std::vector<int> cl(B, ctx), nr(B, N), par;
        for (int b = 0; b < B; ++b) {
            std::vector<int> dep(N, 0);
            for (int i = 0; i < N; ++i) {
                int p = i == 0 ? -1 : (i - 1) / 10;
                if (i) {
                    while (dep[p] + 1 >= sgb::kMaxChain) p = (p - 1) / 10;
                    dep[i] = dep[p] + 1;
                }
                par.push_back(p);
            }
        }
        TreeAttnCase c(B, cl.data(), nr.data(), par.data(), H, dh, nullptr, nullptr, nullptr, nullptr, nullptr);
        cudaEvent_t a, b;
        SGB_CUDA(cudaEventCreate(&a));
        SGB_CUDA(cudaEventCreate(&b));
        float ms = 0.f;
        for (int pass = 0; pass < 2; ++pass) {
            for (int i = 0; i < 2; ++i) pass ? c.run_group() : c.run_row();
            SGB_CUDA(cudaEventRecord(a, 0));
            for (int i = 0; i < iters; ++i) pass ? c.run_group() : c.run_row();
            SGB_CUDA(cudaEventRecord(b, 0));
            SGB_CUDA(cudaEventSynchronize(b));
            SGB_CUDA(cudaEventElapsedTime(&ms, a, b));
            (pass ? *ms_group : *ms_row) = ms / iters;
        }
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    });
}

// Decode-attention microbenchmark: B sequences x H heads, each one query row attending to
// ctx cached keys + itself (AR decode shape), KV in a [B*(ctx+1)][d] bf16 store.
int sgb_bench_attention(int B, int ctx, int H, int dh, int iters, double* ms_out) {
    return guarded([&] {
        const int d = H * dh;
        const long long slots = static_cast<long long>(B) * (ctx + 1);
        __nv_bfloat16 *K = nullptr, *V = nullptr, *out = nullptr;
        float *q = nullptr, *pacc = nullptr, *pml = nullptr;
        SGB_CUDA(cudaMalloc(&K, slots * d * 2));
        SGB_CUDA(cudaMalloc(&V, slots * d * 2));
        SGB_CUDA(cudaMemset(K, 0x3c, slots * d * 2));
        SGB_CUDA(cudaMemset(V, 0x3c, slots * d * 2));
        SGB_CUDA(cudaMalloc(&q, static_cast<size_t>(B) * d * 4));
        SGB_CUDA(cudaMemset(q, 0, static_cast<size_t>(B) * d * 4));
        SGB_CUDA(cudaMalloc(&out, static_cast<size_t>(B) * d * 2));
        const int ns = sgb::attn_splits_for(ctx + 1);
        SGB_CUDA(cudaMalloc(&pacc, static_cast<size_t>(B) * d * ns * 4));
        SGB_CUDA(cudaMalloc(&pml, static_cast<size_t>(B) * H * ns * 2 * 4));
        std::vector<long long> base(B), chain(static_cast<size_t>(B) * sgb::kMaxChain, 0);
        std::vector<int> cl(B, ctx), chl(B, 1);
        for (int b = 0; b < B; ++b) {
            base[b] = static_cast<long long>(b) * (ctx + 1);
            chain[static_cast<size_t>(b) * sgb::kMaxChain] = base[b] + ctx;
        }
        long long *dbase = nullptr, *dchain = nullptr;
        int *dcl = nullptr, *dchl = nullptr;
        SGB_CUDA(cudaMalloc(&dbase, B * 8));
        SGB_CUDA(cudaMalloc(&dchain, chain.size() * 8));
        SGB_CUDA(cudaMalloc(&dcl, B * 4));
        SGB_CUDA(cudaMalloc(&dchl, B * 4));
        SGB_CUDA(cudaMemcpy(dbase, base.data(), B * 8, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dchain, chain.data(), chain.size() * 8, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dcl, cl.data(), B * 4, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dchl, chl.data(), B * 4, cudaMemcpyHostToDevice));
        sgb::AttnRowsDev ar{dbase, dcl, dchl, dchain};
        sgb::AttnScratch sc{pacc, pml, nullptr, static_cast<long long>(B) * H};
        SGB_CUDA(cudaMalloc(&sc.row_ctr, sc.ctr_cap * 4));
        SGB_CUDA(cudaMemset(sc.row_ctr, 0, sc.ctr_cap * 4));
        const double keys = static_cast<double>(B) * (ctx + 1);
        cudaEvent_t a, b;
        SGB_CUDA(cudaEventCreate(&a));
        SGB_CUDA(cudaEventCreate(&b));
        for (int i = 0; i < 2; ++i) sgb::launch_attention(q, K, V, slots, ar, B, H, d, ctx + 1, keys, sc, out, 0);
        SGB_CUDA(cudaEventRecord(a, 0));
        for (int i = 0; i < iters; ++i) sgb::launch_attention(q, K, V, slots, ar, B, H, d, ctx + 1, keys, sc, out, 0);
        SGB_CUDA(cudaEventRecord(b, 0));
        SGB_CUDA(cudaEventSynchronize(b));
        float ms = 0.f;
        SGB_CUDA(cudaEventElapsedTime(&ms, a, b));
        *ms_out = ms / iters;
        void* ptrs[] = {K, V, out, q, pacc, pml, dbase, dchain, dcl, dchl, sc.row_ctr};
        for (void* p : ptrs) cudaFree(p);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
    });
}

int sgb_debug_gemm(const float* w, const float* x, int M, int N, int K, float* out, int* splits_out) {
    return guarded([&] {
        if (M <= 0 || N <= 0 || K <= 0) throw std::invalid_argument("debug_gemm: bad shape");
        std::vector<__nv_bfloat16> wb(static_cast<size_t>(N) * K), xb(static_cast<size_t>(M) * K);
        for (size_t i = 0; i < wb.size(); ++i) wb[i] = __float2bfloat16(w[i]);
        for (size_t i = 0; i < xb.size(); ++i) xb[i] = __float2bfloat16(x[i]);
        __nv_bfloat16 *dw = nullptr, *dx = nullptr;
        float* dp = nullptr;
        const int cap = ((M + 255) / 256) * 256;
        SGB_CUDA(cudaMalloc(&dw, wb.size() * 2));
        SGB_CUDA(cudaMalloc(&dx, static_cast<size_t>(cap) * K * 2));
        SGB_CUDA(cudaMemset(dx, 0, static_cast<size_t>(cap) * K * 2));
        SGB_CUDA(cudaMemcpy(dw, wb.data(), wb.size() * 2, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dx, xb.data(), xb.size() * 2, cudaMemcpyHostToDevice));
        sgb::GemmWeight gw;
        gw.init(dw, N, K);
        sgb::GemmAct ga;
        ga.init(dx, cap, K);
        sgb::GemmWorkspace ws;
        ws.cap_floats = sgb::gemm_ws_floats(M, N, K);
        ws.ctr_cap = 1 << 14;
        SGB_CUDA(cudaMalloc(&ws.buf, ws.cap_floats * 4));
        SGB_CUDA(cudaMalloc(&ws.ctr, ws.ctr_cap * sizeof(int)));
        SGB_CUDA(cudaMemset(ws.ctr, 0, ws.ctr_cap * sizeof(int)));
        SGB_CUDA(cudaMalloc(&dp, static_cast<size_t>(M) * N * 4));
        sgb::GemmEpi epi;
        epi.kind = sgb::kEpiF32;
        epi.f32 = dp;
        epi.ld = N;
        sgb::gemm_run(gw, ga, M, epi, ws, 0, splits_out ? *splits_out : 0);
        SGB_KCHECK();
        SGB_CUDA(cudaDeviceSynchronize());
        SGB_CUDA(cudaMemcpy(out, dp, static_cast<size_t>(M) * N * 4, cudaMemcpyDeviceToHost));
        if (splits_out) *splits_out = sgb::gemm_splits_for(M, N, K);
        cudaFree(ws.buf);
        cudaFree(ws.ctr);
        cudaFree(dw);
        cudaFree(dx);
        cudaFree(dp);
    });
}

}  // extern "C"

// Concurrency microbenchmark for the two-lane AR step: one decoder layer's attention
// (B rows x (ctx + 1) keys, H heads of dh) on one stream and the layer's four GEMMs at M rows
// (QKV, wo, w1, w2 of width d = H*dh and d_ff) on another, each on a capped persistent grid
// (attn_cap / gemm_cap SMs, 0 = all). out[0..2] = ms per iteration: attention alone, GEMMs
// alone, both streams concurrently.
int sgb_bench_overlap(int B, int ctx, int H, int dh, int dff, int M, int attn_cap, int gemm_cap, int iters,
                      double* out) {
    return guarded([&] {
        if (B <= 0 || M <= 0 || iters <= 0) throw std::invalid_argument("bench_overlap: bad shape");
        const int d = H * dh;
        const long long slots = static_cast<long long>(B) * (ctx + 1);
        std::vector<void*> frees;
        auto dmal = [&](size_t bytes) {
            void* p = nullptr;
            SGB_CUDA(cudaMalloc(&p, bytes));
            SGB_CUDA(cudaMemset(p, 0, bytes));
            frees.push_back(p);
            return p;
        };
        auto* K = static_cast<__nv_bfloat16*>(dmal(slots * d * 2));
        auto* V = static_cast<__nv_bfloat16*>(dmal(slots * d * 2));
        SGB_CUDA(cudaMemset(K, 0x3c, slots * d * 2));
        SGB_CUDA(cudaMemset(V, 0x3c, slots * d * 2));
        auto* q = static_cast<float*>(dmal(static_cast<size_t>(B) * d * 4));
        auto* ao = static_cast<__nv_bfloat16*>(dmal(static_cast<size_t>(B) * d * 2));
        const int ns = sgb::attn_splits_for(ctx + 1);
        sgb::AttnScratch sc{static_cast<float*>(dmal(static_cast<size_t>(B) * d * ns * 4)),
                            static_cast<float*>(dmal(static_cast<size_t>(B) * H * ns * 8)), nullptr,
                            static_cast<long long>(B) * H};
        sc.row_ctr = static_cast<int*>(dmal(sc.ctr_cap * 4));
        std::vector<long long> base(B), chain(static_cast<size_t>(B) * sgb::kMaxChain, 0);
        std::vector<int> cl(B, ctx), chl(B, 1);
        for (int b = 0; b < B; ++b) {
            base[b] = static_cast<long long>(b) * (ctx + 1);
            chain[static_cast<size_t>(b) * sgb::kMaxChain] = base[b] + ctx;
        }
        auto* dbase = static_cast<long long*>(dmal(B * 8));
        auto* dchain = static_cast<long long*>(dmal(chain.size() * 8));
        auto* dcl = static_cast<int*>(dmal(B * 4));
        auto* dchl = static_cast<int*>(dmal(B * 4));
        SGB_CUDA(cudaMemcpy(dbase, base.data(), B * 8, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dchain, chain.data(), chain.size() * 8, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dcl, cl.data(), B * 4, cudaMemcpyHostToDevice));
        SGB_CUDA(cudaMemcpy(dchl, chl.data(), B * 4, cudaMemcpyHostToDevice));
        sgb::AttnRowsDev ar{dbase, dcl, dchl, dchain};
        const double keys = static_cast<double>(B) * (ctx + 1);
        // the layer's GEMMs, weights in rotating copies (> L2) as in the rollout
        const int shp[4][2] = {{3 * d, d}, {d, d}, {dff, d}, {d, dff}};
        const int ncopy = 4;
        std::vector<sgb::GemmWeight> gw(4 * ncopy);
        for (int g = 0; g < 4; ++g)
            for (int c = 0; c < ncopy; ++c) {
                auto* w = static_cast<__nv_bfloat16*>(dmal(static_cast<size_t>(shp[g][0]) * shp[g][1] * 2));
                gw[g * ncopy + c].init(w, shp[g][0], shp[g][1]);
            }
        const int cap = ((M + 255) / 256) * 256;
        auto* xa = static_cast<__nv_bfloat16*>(dmal(static_cast<size_t>(cap) * std::max(d, dff) * 2));
        sgb::GemmAct act_d, act_f;
        act_d.init(xa, cap, d);
        act_f.init(xa, cap, dff);
        auto* yo = static_cast<float*>(dmal(static_cast<size_t>(M) * 3 * std::max(d, dff) * 4));
        sgb::GemmWorkspace ws;
        sgb::GemmEpi epi;
        epi.kind = sgb::kEpiF32;
        epi.f32 = yo;
        cudaStream_t s1, s2;
        SGB_CUDA(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
        SGB_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        cudaEvent_t a, b, j;
        SGB_CUDA(cudaEventCreate(&a));
        SGB_CUDA(cudaEventCreate(&b));
        SGB_CUDA(cudaEventCreate(&j));
        int rot = 0;
        auto attn = [&] {
            sgb::g_attn_sm_cap = attn_cap;
            sgb::launch_attention(q, K, V, slots, ar, B, H, d, ctx + 1, keys, sc, ao, s1);
            sgb::g_attn_sm_cap = 0;
        };
        auto gemms = [&] {
            sgb::g_gemm_sm_cap = gemm_cap;
            for (int g = 0; g < 4; ++g) {
                epi.ld = shp[g][0];
                sgb::gemm_run(gw[g * ncopy + rot % ncopy], g == 3 ? act_f : act_d, M, epi, ws, s2, 1);
            }
            ++rot;
            sgb::g_gemm_sm_cap = 0;
        };
        auto time = [&](bool ra, bool rg) {
            for (int w = 0; w < 2; ++w) {
                if (ra) attn();
                if (rg) gemms();
            }
            SGB_CUDA(cudaDeviceSynchronize());
            SGB_CUDA(cudaEventRecord(a, s1));
            SGB_CUDA(cudaStreamWaitEvent(s2, a, 0));
            for (int i = 0; i < iters; ++i) {
                if (ra) attn();
                if (rg) gemms();
            }
            SGB_CUDA(cudaEventRecord(j, s2));
            SGB_CUDA(cudaStreamWaitEvent(s1, j, 0));
            SGB_CUDA(cudaEventRecord(b, s1));
            SGB_CUDA(cudaEventSynchronize(b));
            SGB_KCHECK();
            float ms = 0.f;
            SGB_CUDA(cudaEventElapsedTime(&ms, a, b));
            return static_cast<double>(ms) / iters;
        };
        out[0] = time(true, false);
        out[1] = time(false, true);
        out[2] = time(true, true);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaEventDestroy(j);
        cudaStreamDestroy(s1);
        cudaStreamDestroy(s2);
        for (void* p : frees) cudaFree(p);
    });
}
