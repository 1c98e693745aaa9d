// Engine: device weights, KV stores, batched forward passes and the rollout step loop.
//
// The rollout is generate_dynamic_batch (src/scheduler.cpp:236-354) restated for a GPU:
// the reference runs one forward per *sequence* per step (scheduler.cpp:322-328); here one
// step is ONE batched target forward over the flattened trees of all live sequences, plus
// one batched draft catch-up forward and (L-1) batched draft-level forwards. All tree
// decisions run in device kernels (tree.cu); the host only plans the step (Eqs. 1-3,
// scheduler.cpp:14-54 -- pure integer work that needs the live count B_cur) and reads back
// one small per-sequence result vector per step.
#include <algorithm>
#include <chrono>
#include <optional>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <cmath>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <string>

#include "common.cuh"
#include "engine.h"
#include "util.h"

namespace sgb {

namespace {


template <class T>
T* dalloc(size_t n) {
    T* p = nullptr;
    if (n == 0) n = 1;
    SGB_CUDA(cudaMalloc(&p, n * sizeof(T)));
    return p;
}

template <class T>
void h2d(T* dst, const T* src, size_t n, cudaStream_t st) {
    if (n) SGB_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, st));
}
template <class T>
void d2h(T* dst, const T* src, size_t n, cudaStream_t st) {
    if (n) SGB_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, st));
}

int tree_cap(int k, int l) { return 1 + k + std::max(0, l - 1) * k * k; }  // drafttree.cpp:11-15

// Eqs. 1-3 (scheduler.cpp:26-54).
SpecCfg plan(int c_peak, int b, double alpha, int k_max, int l_max) {
    if (c_peak < 1 || b < 1) throw std::invalid_argument("compute_n_verify: c_peak, b >= 1");
    if (alpha <= 0) throw std::invalid_argument("compute_l_draft: alpha must be positive");
    SpecCfg c;
    c.n_verify = std::max(1, c_peak / b);
    c.k_draft = std::max(0, std::min(c.n_verify - 1, k_max));
    if (c.k_draft == 0) {
        c.l_draft = 0;
    } else {
        const int raw = static_cast<int>(std::floor(std::log2(static_cast<double>(c.n_verify) / alpha)));
        c.l_draft = std::max(1, std::min(raw, l_max));
    }
    if (c.l_draft > l_max) throw std::invalid_argument("spec config: l_draft exceeds l_max");
    return c;
}

void validate_spec(const SpecCfg& c, double alpha, int k_max, int l_max, int c_peak) {  // scheduler.cpp:14-24
    if (c.n_verify < 1) throw std::invalid_argument("spec config: n_verify must be >= 1");
    if (c.k_draft < 0 || c.l_draft < 0) throw std::invalid_argument("spec config: k_draft/l_draft must be >= 0");
    if (c.k_draft > std::max(0, c.n_verify - 1))
        throw std::invalid_argument("spec config: k_draft must be <= n_verify - 1");
    if (c.k_draft > k_max) throw std::invalid_argument("spec config: k_draft exceeds k_max");
    if (c.l_draft > l_max) throw std::invalid_argument("spec config: l_draft exceeds l_max");
    if (alpha <= 0) throw std::invalid_argument("spec config: alpha must be positive");
    if (c_peak < 1) throw std::invalid_argument("spec config: c_peak must be >= 1");
}

uint64_t splitmix_host(uint64_t& s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
uint64_t mix_key_host(uint64_t a, uint64_t b) {  // rng.hpp:17-20
    uint64_t s = a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2));
    return splitmix_host(s);
}

}  // namespace

// ------------------------------------------------------------------ layouts
FlatLayout FlatLayout::target(const ModelDims& m) {
    FlatLayout f;
    size_t o = 0;
    const size_t d = m.d;
    auto add = [&](size_t n) {
        size_t r = o;
        o += n;
        return r;
    };
    f.tok_emb = add(static_cast<size_t>(m.vocab) * d);
    f.pos_emb = add(static_cast<size_t>(m.max_seq) * d);
    for (int l = 0; l < m.layers; ++l) {
        L x;
        x.ln1_g = add(d);
        x.ln1_b = add(d);
        x.wq = add(d * d);
        x.wk = add(d * d);
        x.wv = add(d * d);
        x.wo = add(d * d);
        x.ln2_g = add(d);
        x.ln2_b = add(d);
        x.w1 = add(d * m.dff);
        x.w2 = add(d * m.dff);
        f.layers.push_back(x);
    }
    f.lnf_g = add(d);
    f.lnf_b = add(d);
    f.lm_head = add(d * m.vocab);
    f.total = o;
    return f;
}

FlatLayout FlatLayout::draft(const ModelDims& m, int n_layers) {
    FlatLayout f;
    size_t o = 0;
    const size_t d = m.d;
    auto add = [&](size_t n) {
        size_t r = o;
        o += n;
        return r;
    };
    f.w_fuse = add(2 * d * d);
    for (int l = 0; l < n_layers; ++l) {
        L x;
        x.ln1_g = add(d);
        x.ln1_b = add(d);
        x.wq = add(d * d);
        x.wk = add(d * d);
        x.wv = add(d * d);
        x.wo = add(d * d);
        x.ln2_g = add(d);
        x.ln2_b = add(d);
        x.w1 = add(d * m.dff);
        x.w2 = add(d * m.dff);
        f.layers.push_back(x);
    }
    f.lnf_g = add(d);
    f.lnf_b = add(d);
    f.total = o;
    return f;
}

// ------------------------------------------------------------------ construction
Engine::Engine(const ModelDims& dims, int draft_layers, int device, int max_seqs, int max_rows, int k_max, int l_max)
    : dims_(dims), dlayers_(draft_layers), device_(device), max_seqs_(max_seqs), k_max_(k_max), l_max_(l_max) {
    if (dims.vocab < 4 || dims.d <= 0 || dims.layers <= 0 || dims.heads <= 0 || dims.dff <= 0)
        throw std::invalid_argument("model dims must be positive (vocab >= 4)");
    if (dims.d % dims.heads) throw std::invalid_argument("d_model must be divisible by n_heads");
    if (dims.max_seq < 8) throw std::invalid_argument("max_seq_len must be >= 8");
    const int dh = dims.d / dims.heads;
    if (dh != 64 && dh != 128 && dh != 256) throw std::invalid_argument("head dim must be 64, 128 or 256");
    if (dims.d % 8 || dims.dff % 8) throw std::invalid_argument("d_model and d_ff must be multiples of 8");
    if (draft_layers <= 0) throw std::invalid_argument("draft n_layers must be positive");
    if (k_max < 0 || k_max > 16) throw std::invalid_argument("engine k_max must be in [0, 16]");
    if (l_max < 0 || l_max + 1 > kMaxChain) throw std::invalid_argument("engine l_max must be in [0, 7]");
    if (max_seqs < 1) throw std::invalid_argument("max_seqs must be >= 1");
    max_rows_ = std::max(256, ((max_rows + 255) / 256) * 256);
    SGB_CUDA(cudaSetDevice(device));
    SGB_CUDA(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking));
    SGB_CUDA(cudaEventCreate(&ev0_));
    SGB_CUDA(cudaEventCreate(&ev1_));
    SGB_CUDA(cudaEventCreate(&evs_a_));
    SGB_CUDA(cudaEventCreate(&evs_b_));
    SGB_CUDA(cudaEventCreate(&evs_c_));
    tlay_ = FlatLayout::target(dims);
    dlay_ = FlatLayout::draft(dims, draft_layers);

    const size_t d = dims.d, V = dims.vocab, T = dims.max_seq, F = dims.dff, S = max_seqs, R = max_rows_;
    const int ds = 1 + std::max(0, l_max - 1) * std::max(1, k_max);
    // weights
    const size_t per_layer_bf = 4 * d * d + 2 * d * F;
    tw_ = dalloc<__nv_bfloat16>(dims.layers * per_layer_bf + V * d);
    dw_ = dalloc<__nv_bfloat16>(draft_layers * per_layer_bf + 2 * d * d);
    tsmall_ = dalloc<float>(V * d + T * d + dims.layers * 4 * d + 2 * d);
    dmaster_ = dalloc<float>(dlay_.total);
    // KV stores
    tkv_.layers = dims.layers;
    tkv_.seq_stride = T;
    tkv_.scratch_base = static_cast<long long>(S) * T;
    tkv_.n_slots = tkv_.scratch_base + R;
    tkv_.K = dalloc<__nv_bfloat16>(static_cast<size_t>(tkv_.n_slots) * d * dims.layers);
    tkv_.V = dalloc<__nv_bfloat16>(static_cast<size_t>(tkv_.n_slots) * d * dims.layers);
    dkv_.layers = draft_layers;
    dkv_.seq_stride = T;
    dkv_.scratch_base = static_cast<long long>(S) * T;
    dkv_.n_slots = dkv_.scratch_base + static_cast<long long>(S) * ds;
    dkv_.K = dalloc<__nv_bfloat16>(static_cast<size_t>(dkv_.n_slots) * d * draft_layers);
    dkv_.V = dalloc<__nv_bfloat16>(static_cast<size_t>(dkv_.n_slots) * d * draft_layers);
    // every KV slot holds finite values from the start: attention stages whole 16-key boxes and
    // masks the keys past a row's end (p = 0), which must not meet NaN bit patterns
    SGB_CUDA(cudaMemset(tkv_.K, 0, static_cast<size_t>(tkv_.n_slots) * d * dims.layers * 2));
    SGB_CUDA(cudaMemset(tkv_.V, 0, static_cast<size_t>(tkv_.n_slots) * d * dims.layers * 2));
    SGB_CUDA(cudaMemset(dkv_.K, 0, static_cast<size_t>(dkv_.n_slots) * d * draft_layers * 2));
    SGB_CUDA(cudaMemset(dkv_.V, 0, static_cast<size_t>(dkv_.n_slots) * d * draft_layers * 2));
    tkmap_ = make_kmajor_map(tkv_.K, static_cast<int>(tkv_.n_slots * dims.layers), static_cast<int>(d), 16);
    tvmap_ = make_kmajor_map(tkv_.V, static_cast<int>(tkv_.n_slots * dims.layers), static_cast<int>(d), 16);
    dkmap_ = make_kmajor_map(dkv_.K, static_cast<int>(dkv_.n_slots * draft_layers), static_cast<int>(d), 16);
    dvmap_ = make_kmajor_map(dkv_.V, static_cast<int>(dkv_.n_slots * draft_layers), static_cast<int>(d), 16);
    // sequences
    ss_.max_seq = static_cast<int>(T);
    ss_.tokens = dalloc<int>(S * T);
    ss_.len = dalloc<int>(S);
    ss_.finished = dalloc<int>(S);
    ss_.hit_eos = dalloc<int>(S);
    ss_.seed = dalloc<unsigned long long>(S);
    feats_ = dalloc<float>(S * T * d);
    dfeat_ = dalloc<float>(S * ds * d);
    tr_.tmax = tree_cap(std::max(1, k_max), std::max(1, l_max));
    if (tr_.tmax > 1024) throw std::invalid_argument("tree capacity exceeds 1024 nodes (k_max, l_max too large)");
    tr_.ds = ds;
    const size_t TM = static_cast<size_t>(tr_.tmax) * S;
    tr_.tok = dalloc<int>(TM);
    tr_.par = dalloc<int>(TM);
    tr_.dep = dalloc<int>(TM);
    tr_.lp = dalloc<double>(TM);
    tr_.conf = dalloc<double>(TM);
    tr_.fslot = dalloc<int>(TM);
    tr_.sel = dalloc<int>(TM);
    tr_.n_nodes = dalloc<int>(S);
    tr_.lvl_start = dalloc<int>(S);
    tr_.lvl_cnt = dalloc<int>(S);
    tr_.frontier = dalloc<int>(S * 16);
    cache_len_t_.assign(S, 0);
    cache_len_d_.assign(S, 0);
    // activations
    x_ = dalloc<float>(R * d);
    q_ = dalloc<float>(R * d);
    y_ = dalloc<float>(R * d);
    featin_ = dalloc<float>(R * d);
    a_ = dalloc<__nv_bfloat16>(R * d);
    att_ = dalloc<__nv_bfloat16>(R * d);
    a2_ = dalloc<__nv_bfloat16>(R * d);
    h_ = dalloc<__nv_bfloat16>(R * F);
    fuse_ = dalloc<__nv_bfloat16>(R * 2 * d);
    act_a_.init(a_, static_cast<int>(R), static_cast<int>(d));
    act_att_.init(att_, static_cast<int>(R), static_cast<int>(d));
    act_a2_.init(a2_, static_cast<int>(R), static_cast<int>(d));
    act_h_.init(h_, static_cast<int>(R), static_cast<int>(F));
    act_fuse_.init(fuse_, static_cast<int>(R), static_cast<int>(2 * d));
    ws_.cap_floats = static_cast<size_t>(64) << 20;  // 256 MiB split-K workspace
    ws_.buf = dalloc<float>(ws_.cap_floats);
    ws_.ctr_cap = 1 << 16;
    ws_.ctr = dalloc<int>(ws_.ctr_cap);
    SGB_CUDA(cudaMemset(ws_.ctr, 0, sizeof(int) * ws_.ctr_cap));
    logits_ = dalloc<float>(R * V);
    {
        int ncmax = std::max(gemm_chunks(static_cast<int>(d), static_cast<int>(d)),
                             gemm_chunks(static_cast<int>(d), static_cast<int>(F)));
        ncmax = std::max(ncmax, gemm_chunks(static_cast<int>(d), static_cast<int>(2 * d)));
        gpart_cap_ = static_cast<size_t>(ncmax) * R * d;
        gpart_ = dalloc<float>(gpart_cap_);
    }
    rsc_.rows = static_cast<int>(R);
    rsc_.bytes = row_scratch_bytes(static_cast<int>(R), static_cast<int>(V));
    rsc_.buf = dalloc<unsigned char>(rsc_.bytes);
    rsc_.ctr = dalloc<int>(R);
    rsc_.rowmax = dalloc<float>(R);
    rsc_.exact = dalloc<int>(R);
    rsc_.n_exact = dalloc<unsigned long long>(1);
    SGB_CUDA(cudaMemset(rsc_.ctr, 0, sizeof(int) * R));
    SGB_CUDA(cudaMemset(rsc_.exact, 0, sizeof(int) * R));
    SGB_CUDA(cudaMemset(rsc_.n_exact, 0, sizeof(unsigned long long)));
    max_vlen_cap_ = static_cast<int>(T) + kMaxChain;
    const int ns = attn_splits_for(max_vlen_cap_);
    pacc_ = dalloc<float>(R * d * ns);
    pml_ = dalloc<float>(R * dims.heads * ns * 2);
    asc_.part_acc = pacc_;
    asc_.part_ml = pml_;
    asc_.ctr_cap = static_cast<long long>(R) * dims.heads;
    asc_.row_ctr = dalloc<int>(asc_.ctr_cap);
    SGB_CUDA(cudaMemset(asc_.row_ctr, 0, sizeof(int) * asc_.ctr_cap));
    alloc_rows();
    SGB_CUDA(cudaMallocHost(&h_result_, sizeof(int) * (2 * S + 4)));
    SGB_CUDA(cudaMemset(err_, 0, sizeof(int)));
    SGB_CUDA(cudaDeviceSynchronize());
}

void Engine::alloc_rows() {
    const size_t R = max_rows_, S = max_seqs_;
    rows_.tok = dalloc<int>(R);
    rows_.pos = dalloc<int>(R);
    rows_.kv_dst = dalloc<long long>(R);
    rows_.ctx_base = dalloc<long long>(R);
    rows_.ctx_len = dalloc<int>(R);
    rows_.chain_len = dalloc<int>(R);
    rows_.chain = dalloc<long long>(R * kMaxChain);
    rows_.feat_off = dalloc<long long>(R);
    rows_.out_off = dalloc<long long>(R);
    rows_.key_pos = dalloc<int>(R);
    rows_.seed = dalloc<unsigned long long>(R);
    rows_.par_row = dalloc<int>(R);
    rows_.pre_base = dalloc<long long>(R);
    rows_.pre_len = dalloc<int>(R);
    lm_idx_ = dalloc<int>(R);
    topk_tok_ = dalloc<int>(R * 16);
    topk_lp_ = dalloc<double>(R * 16);
    emitted_ = dalloc<int>(R);
    acc_rows_ = dalloc<int>(S * kMaxChain);
    result_ = dalloc<int>(2 * S);
    err_ = dalloc<int>(1);
    steps_ = dalloc<StepSeqDev>(S);
    tiles_ = dalloc<AttnTileDev>(2 * R);
    d_tgroups_ = dalloc<TreeGroupDev>(S + R);
    d_ttiles_ = dalloc<TreeTileDev>(S + R);
    drow_ = dalloc<int>(S * std::max(1, l_max_));
    misc_i_ = dalloc<int>(4 * R + 4 * S);
    misc_l_ = dalloc<long long>(2 * R + 2 * S);
    mask_dbg_ = dalloc<unsigned char>(1024 * 1024);
}

Engine::~Engine() {
    cudaSetDevice(device_);
    cudaStreamSynchronize(st_);
    if (adv_buf_) cudaFree(adv_buf_);
    for (void* q : pol_ptrs_) cudaFree(q);
    if (tmaster_) cudaFree(tmaster_);
    for (void* q : {static_cast<void*>(qbuf_), static_cast<void*>(qstat_), 
                    static_cast<void*>(rkeys_), static_cast<void*>(tr_.qrow)})
        if (q) cudaFree(q);
    void* ptrs[] = {tw_, dw_, tsmall_, dmaster_, tkv_.K, tkv_.V, dkv_.K, dkv_.V, ss_.tokens, ss_.len, ss_.finished,
                    ss_.hit_eos, ss_.seed, feats_, dfeat_, tr_.tok, tr_.par, tr_.dep, tr_.lp, tr_.conf, tr_.fslot,
                    tr_.sel, tr_.n_nodes, tr_.lvl_start, tr_.lvl_cnt, tr_.frontier, x_, q_, y_, featin_, a_, att_,
                    a2_, h_, fuse_, ws_.buf, ws_.ctr, logits_, pacc_, pml_, rows_.tok, rows_.pos, rows_.kv_dst,
                    rows_.ctx_base, rows_.ctx_len, rows_.chain_len, rows_.chain, rows_.feat_off, rows_.out_off,
                    rows_.key_pos, rows_.seed, rows_.par_row, rows_.pre_base, rows_.pre_len, lm_idx_, topk_tok_, topk_lp_, emitted_, acc_rows_,
                    result_, err_, steps_, drow_, misc_i_, misc_l_, mask_dbg_, d_tgroups_, d_ttiles_, rsc_.buf, rsc_.ctr, rsc_.rowmax, rsc_.exact, rsc_.n_exact, asc_.row_ctr, gpart_};
    for (void* p : ptrs)
        if (p) cudaFree(p);
    if (h_result_) cudaFreeHost(h_result_);
    if (feats_host_) cudaFreeHost(feats_host_);
    if (ev0_) cudaEventDestroy(ev0_);
    if (ev1_) cudaEventDestroy(ev1_);
    if (evs_a_) cudaEventDestroy(evs_a_);
    if (evs_b_) cudaEventDestroy(evs_b_);
    if (evs_c_) cudaEventDestroy(evs_c_);
    if (st_) cudaStreamDestroy(st_);
}

// ------------------------------------------------------------------ weights
void Engine::convert_target(const float* stg) {
    const int d = dims_.d, F = dims_.dff, V = dims_.vocab, T = dims_.max_seq;
    float* sm = tsmall_;
    SGB_CUDA(cudaMemcpyAsync(sm, stg + tlay_.tok_emb, sizeof(float) * V * d, cudaMemcpyDeviceToDevice, st_));
    tok_emb_ = sm;
    sm += static_cast<size_t>(V) * d;
    SGB_CUDA(cudaMemcpyAsync(sm, stg + tlay_.pos_emb, sizeof(float) * T * d, cudaMemcpyDeviceToDevice, st_));
    pos_emb_ = sm;
    sm += static_cast<size_t>(T) * d;
    __nv_bfloat16* w = tw_;
    tL_.assign(dims_.layers, LayerDev{});
    for (int l = 0; l < dims_.layers; ++l) {
        const auto& o = tlay_.layers[l];
        LayerDev& L = tL_[l];
        const size_t ln[4] = {o.ln1_g, o.ln1_b, o.ln2_g, o.ln2_b};
        const float** dst[4] = {&L.ln1_g, &L.ln1_b, &L.ln2_g, &L.ln2_b};
        for (int i = 0; i < 4; ++i) {
            SGB_CUDA(cudaMemcpyAsync(sm, stg + ln[i], sizeof(float) * d, cudaMemcpyDeviceToDevice, st_));
            *dst[i] = sm;
            sm += d;
        }
        __nv_bfloat16* qkv = w;
        launch_transpose_to_bf16(stg + o.wq, d, d, qkv, d, st_);
        launch_transpose_to_bf16(stg + o.wk, d, d, qkv + static_cast<size_t>(d) * d, d, st_);
        launch_transpose_to_bf16(stg + o.wv, d, d, qkv + 2 * static_cast<size_t>(d) * d, d, st_);
        w += 3 * static_cast<size_t>(d) * d;
        __nv_bfloat16* wo = w;
        launch_transpose_to_bf16(stg + o.wo, d, d, wo, d, st_);
        w += static_cast<size_t>(d) * d;
        __nv_bfloat16* w1 = w;
        launch_transpose_to_bf16(stg + o.w1, d, F, w1, d, st_);
        w += static_cast<size_t>(d) * F;
        __nv_bfloat16* w2 = w;
        launch_transpose_to_bf16(stg + o.w2, F, d, w2, F, st_);
        w += static_cast<size_t>(d) * F;
        L.qkv.init(qkv, 3 * d, d);
        L.wo.init(wo, d, d);
        L.w1.init(w1, F, d);
        L.w2.init(w2, d, F);
    }
    SGB_CUDA(cudaMemcpyAsync(sm, stg + tlay_.lnf_g, sizeof(float) * d, cudaMemcpyDeviceToDevice, st_));
    lnf_g_ = sm;
    sm += d;
    SGB_CUDA(cudaMemcpyAsync(sm, stg + tlay_.lnf_b, sizeof(float) * d, cudaMemcpyDeviceToDevice, st_));
    lnf_b_ = sm;
    launch_transpose_to_bf16(stg + tlay_.lm_head, d, V, w, d, st_);
    lm_head_.init(w, V, d);
    SGB_CUDA(cudaStreamSynchronize(st_));
    target_ready_ = true;
}

void Engine::convert_draft() {
    const int d = dims_.d, F = dims_.dff;
    const float* m = dmaster_;
    __nv_bfloat16* w = dw_;
    launch_transpose_to_bf16(m + dlay_.w_fuse, 2 * d, d, w, 2 * d, st_);
    w_fuse_.init(w, d, 2 * d);
    w += 2 * static_cast<size_t>(d) * d;
    dL_.assign(dlayers_, LayerDev{});
    for (int l = 0; l < dlayers_; ++l) {
        const auto& o = dlay_.layers[l];
        LayerDev& L = dL_[l];
        L.ln1_g = m + o.ln1_g;
        L.ln1_b = m + o.ln1_b;
        L.ln2_g = m + o.ln2_g;
        L.ln2_b = m + o.ln2_b;
        __nv_bfloat16* qkv = w;
        launch_transpose_to_bf16(m + o.wq, d, d, qkv, d, st_);
        launch_transpose_to_bf16(m + o.wk, d, d, qkv + static_cast<size_t>(d) * d, d, st_);
        launch_transpose_to_bf16(m + o.wv, d, d, qkv + 2 * static_cast<size_t>(d) * d, d, st_);
        w += 3 * static_cast<size_t>(d) * d;
        __nv_bfloat16* wo = w;
        launch_transpose_to_bf16(m + o.wo, d, d, wo, d, st_);
        w += static_cast<size_t>(d) * d;
        __nv_bfloat16* w1 = w;
        launch_transpose_to_bf16(m + o.w1, d, F, w1, d, st_);
        w += static_cast<size_t>(d) * F;
        __nv_bfloat16* w2 = w;
        launch_transpose_to_bf16(m + o.w2, F, d, w2, F, st_);
        w += static_cast<size_t>(d) * F;
        L.qkv.init(qkv, 3 * d, d);
        L.wo.init(wo, d, d);
        L.w1.init(w1, F, d);
        L.w2.init(w2, d, F);
    }
    dlnf_g_ = m + dlay_.lnf_g;
    dlnf_b_ = m + dlay_.lnf_b;
    SGB_CUDA(cudaStreamSynchronize(st_));
    draft_ready_ = true;
}

void Engine::upload_target(const float* flat, size_t n) {
    if (n != tlay_.total) throw std::invalid_argument("upload_target: param count mismatch");
    float* stg = tmaster_ ? tmaster_ : dalloc<float>(n);
    SGB_CUDA(cudaMemcpy(stg, flat, n * sizeof(float), cudaMemcpyHostToDevice));
    convert_target(stg);
    draft_lm_stale_ = tr2_.ready;  // the draft update's frozen copy of the LM head
    if (keep_master_) {
        tmaster_ = stg;  // the policy update's fp32 master
        if (pol_.ready) policy_refresh_ref_weights();
    } else {
        cudaFree(stg);
    }
}

void Engine::upload_draft(const float* flat, size_t n) {
    if (n != dlay_.total) throw std::invalid_argument("upload_draft: param count mismatch");
    SGB_CUDA(cudaMemcpy(dmaster_, flat, n * sizeof(float), cudaMemcpyHostToDevice));
    convert_draft();
}

void Engine::download_draft(float* flat, size_t n) {
    if (n != dlay_.total) throw std::invalid_argument("download_draft: param count mismatch");
    SGB_CUDA(cudaStreamSynchronize(st_));
    SGB_CUDA(cudaMemcpy(flat, dmaster_, n * sizeof(float), cudaMemcpyDeviceToHost));
}

// Same distributions as init_flat (tinylm.hpp:83-109) but drawn by a device counter RNG,
// so large benchmark models initialise in milliseconds (not reference-identical values).
void Engine::init_random(uint64_t seed) {
    const int d = dims_.d, F = dims_.dff, V = dims_.vocab, T = dims_.max_seq;
    float* stg = dalloc<float>(tlay_.total);
    uint64_t s = seed;
    auto nrm = [&](size_t off, size_t n, float sd) { launch_init_normal(stg + off, n, splitmix_host(s), sd, st_); };
    auto one = [&](size_t off, size_t n, float v) { launch_fill(stg + off, n, v, st_); };
    const float res_t = static_cast<float>(0.02 / std::sqrt(2.0 * dims_.layers));
    nrm(tlay_.tok_emb, static_cast<size_t>(V) * d, 0.02f);
    nrm(tlay_.pos_emb, static_cast<size_t>(T) * d, 0.01f);
    for (const auto& o : tlay_.layers) {
        one(o.ln1_g, d, 1.f);
        one(o.ln1_b, d, 0.f);
        one(o.ln2_g, d, 1.f);
        one(o.ln2_b, d, 0.f);
        nrm(o.wq, static_cast<size_t>(d) * d, 0.02f);
        nrm(o.wk, static_cast<size_t>(d) * d, 0.02f);
        nrm(o.wv, static_cast<size_t>(d) * d, 0.02f);
        nrm(o.wo, static_cast<size_t>(d) * d, res_t);
        nrm(o.w1, static_cast<size_t>(d) * F, 0.02f);
        nrm(o.w2, static_cast<size_t>(d) * F, res_t);
    }
    one(tlay_.lnf_g, d, 1.f);
    one(tlay_.lnf_b, d, 0.f);
    nrm(tlay_.lm_head, static_cast<size_t>(d) * V, 0.02f);
    convert_target(stg);
    draft_lm_stale_ = tr2_.ready;
    if (keep_master_) {
        if (tmaster_) cudaFree(tmaster_);
        tmaster_ = stg;
        if (pol_.ready) policy_refresh_ref_weights();
    } else {
        cudaFree(stg);
    }
    const float res_d = static_cast<float>(0.02 / std::sqrt(2.0 * dlayers_));
    float* m = dmaster_;
    launch_init_normal(m + dlay_.w_fuse, 2 * static_cast<size_t>(d) * d, splitmix_host(s), 0.02f, st_);
    for (const auto& o : dlay_.layers) {
        launch_fill(m + o.ln1_g, d, 1.f, st_);
        launch_fill(m + o.ln1_b, d, 0.f, st_);
        launch_fill(m + o.ln2_g, d, 1.f, st_);
        launch_fill(m + o.ln2_b, d, 0.f, st_);
        launch_init_normal(m + o.wq, static_cast<size_t>(d) * d, splitmix_host(s), 0.02f, st_);
        launch_init_normal(m + o.wk, static_cast<size_t>(d) * d, splitmix_host(s), 0.02f, st_);
        launch_init_normal(m + o.wv, static_cast<size_t>(d) * d, splitmix_host(s), 0.02f, st_);
        launch_init_normal(m + o.wo, static_cast<size_t>(d) * d, splitmix_host(s), res_d, st_);
        launch_init_normal(m + o.w1, static_cast<size_t>(d) * F, splitmix_host(s), 0.02f, st_);
        launch_init_normal(m + o.w2, static_cast<size_t>(d) * F, splitmix_host(s), res_d, st_);
    }
    launch_fill(m + dlay_.lnf_g, d, 1.f, st_);
    launch_fill(m + dlay_.lnf_b, d, 0.f, st_);
    convert_draft();
}

// ------------------------------------------------------------------ forward
void Engine::lm_head(const __nv_bfloat16*, const GemmAct& act, int R, float* out) {
    GemmEpi e;
    e.kind = kEpiF32;
    e.f32 = out;
    e.ld = dims_.vocab;
    gemm(lm_head_, act, R, e, kClsLmHead, 4.0);
}

void Engine::gemm(const GemmWeight& w, const GemmAct& a, int M, const GemmEpi& epi, int cls, double out_bytes) {
    const int e0 = pbeg();
    gemm_run(w, a, M, epi, ws_, st_, force_splits_);
    pend(cls, e0, 2.0 * w.N * w.K + 2.0 * M * w.K + out_bytes * M * w.N, 2.0 * M * w.N * w.K);
    count();
}

void Engine::ln(int M, const float* g, const float* b, float* y) {
    const int e0 = pbeg();
    launch_reduce_residual_ln(nullptr, 0, M, dims_.d, x_, false, nullptr, nullptr, g, b, a_, y, st_);
    pend(kClsRow, e0, static_cast<double>(M) * dims_.d * (4 + 2 + (y ? 4 : 0)), 0);
    count();
}

void Engine::gemm_resid_ln(const GemmWeight& w, const GemmAct& a, int M, bool accumulate, bool add_pos,
                           const float* g, const float* b, float* y) {
    const int d = dims_.d;
    const int nc = gemm_chunks(w.N, w.K);
    if (gemm_bn_for(M) >= 64 && nc > 1 && static_cast<size_t>(nc) * M * d <= gpart_cap_) {
        GemmEpi e;
        e.kind = kEpiPartials;
        e.f32 = gpart_;
        e.ld = d;
        gemm(w, a, M, e, kClsGemm, 4.0 * nc);
        const int e0 = pbeg();
        launch_reduce_residual_ln(gpart_, nc, M, d, x_, accumulate, add_pos ? pos_emb_ : nullptr,
                                  add_pos ? rows_.pos : nullptr, g, b, a_, y, st_);
        pend(kClsRow, e0, static_cast<double>(M) * d * (4.0 * nc + 8 + 2 + (y ? 4 : 0)), 0);
        count();
        return;
    }
    GemmEpi e;
    e.kind = add_pos ? kEpiFusePos : kEpiResid;
    e.f32 = x_;
    e.ld = d;
    if (add_pos) {
        e.pos_emb = pos_emb_;
        e.pos = rows_.pos;
    }
    if (!accumulate && !add_pos) throw std::logic_error("gemm_resid_ln: plain store unsupported");
    gemm(w, a, M, e, kClsGemm, 8.0);
    ln(M, g, b, y);
}

// ------------------------------------------------------------------ GRPO rewards / advantages
void Engine::group_advantages(const long long* answers, int n_groups, int g, double eps_var, double* rewards,
                              double* adv, int* valid) {
    const int n = n_groups * g;
    if (n_groups <= 0 || g < 2) throw std::invalid_argument("standardize_advantages: need G >= 2");
    if (last_waves_) throw std::invalid_argument("group_advantages: the last rollout ran in waves (not resident)");
    if (static_cast<size_t>(n) != last_lens_.size()) throw std::invalid_argument("group_advantages: not the last rollout's shape");
    if (n > max_rows_) throw std::invalid_argument("group_advantages: too many sequences");
    int* dlen = misc_i_;
    int* dplen = misc_i_ + n;
    int* dvalid = misc_i_ + 2 * n;
    long long* dans = misc_l_;
    if (!adv_buf_) adv_buf_ = dalloc<double>(2 * static_cast<size_t>(max_rows_));  // n <= max_rows
    double* dbuf = adv_buf_;
    h2d(dlen, last_lens_.data(), n, st_);
    h2d(dplen, last_plens_.data(), n, st_);
    h2d(dans, answers, n_groups, st_);
    launch_group_advantages(n_groups, g, ss_.tokens, dims_.max_seq, dlen, dplen, dans, eps_var, dbuf, dbuf + n, dvalid,
                            st_);
    SGB_CUDA(cudaMemcpyAsync(rewards, dbuf, sizeof(double) * n, cudaMemcpyDeviceToHost, st_));
    SGB_CUDA(cudaMemcpyAsync(adv, dbuf + n, sizeof(double) * n, cudaMemcpyDeviceToHost, st_));
    SGB_CUDA(cudaMemcpyAsync(valid, dvalid, sizeof(int) * n_groups, cudaMemcpyDeviceToHost, st_));
    SGB_CUDA(cudaStreamSynchronize(st_));
}

// Shared-prefix tiles for grouped rows; SGB_ATTN_GROUP=0 runs every row alone (bit-identical,
// for A/B timing), =1 forces tiles for every grouped forward.
static bool group_attn_enabled(int n_groups, int M) {
    static const int mode = [] {
        const char* v = getenv("SGB_ATTN_GROUP");
        return v ? atoi(v) : -1;
    }();
    if (mode == 0 || n_groups <= 0) return false;
    if (mode == 1) return true;
    return M >= 2 * n_groups;
}

// attention_tree.cu for tree verify / draft levels (SGB_TREE_ATTN=0: attention.cu, A/B), when
// the node table of the largest tree fits the kernel's shared memory
bool Engine::tree_attn_ok(int max_nodes) const {
    static const int env = [] {
        const char* v = getenv("SGB_TREE_ATTN");
        return v ? atoi(v) : 1;
    }();
    const int dh = dims_.d / dims_.heads;
    return env != 0 && (dh == 64 || dh == 128) &&
           static_cast<size_t>(max_nodes) * (dh * 2 + 16) * 2 + 4 * 16 * dh * 2 + 2048 <= 227 * 1024;
}

// Prefix-end blocks inside the shared verify / draft-level tiles (attention.cu): measured
// faster at 28 heads (B = 16 x 13 rows, ctx 680: 0.129 -> 0.098 ms per layer), slower at 12
// heads, where fewer head groups leave the longer boundary item on the critical path (0.076 ->
// 0.099 ms; profiles/r01_tree_boundary.txt)
bool Engine::boundary_tiles() const { return dims_.heads > 16; }

void Engine::forward(const Fwd& f) {
    const int M = f.M, d = dims_.d, F = dims_.dff, H = dims_.heads;
    if (M <= 0) return;
    if (M > max_rows_) throw std::invalid_argument("forward: rows exceed engine max_rows");
    if (f.max_vlen > max_vlen_cap_) throw std::out_of_range("forward: context beyond capacity");
    if (!target_ready_ || (f.draft && !draft_ready_)) throw std::runtime_error("weights not uploaded");
    if (!f.draft) ++target_forward_calls_;  // target_forward_calls() (tinylm.hpp:288-291): one per launch
    const std::vector<LayerDev>& L = f.draft ? dL_ : tL_;
    KvStore& kv = f.draft ? dkv_ : tkv_;
    AttnRowsDev ar{rows_.ctx_base, rows_.ctx_len, rows_.chain_len, rows_.chain};
    if (f.prefix_share) {
        ar.pre_base = rows_.pre_base;
        ar.pre_len = rows_.pre_len;
    }
    const double row_bytes = static_cast<double>(M) * d * 4;
    int e0 = pbeg();
    if (!f.draft) {
        launch_embed_ln(rows_.tok, rows_.pos, M, d, tok_emb_, pos_emb_, L[0].ln1_g, L[0].ln1_b, x_, a_, st_);
        pend(kClsRow, e0, 3 * row_bytes, 0);
        count();
    } else {
        launch_gather_fuse(rows_.tok, rows_.feat_off, f.feat_base, tok_emb_, M, d, fuse_, st_);
        pend(kClsRow, e0, 3 * row_bytes, 0);
        count();
        gemm_resid_ln(w_fuse_, act_fuse_, M, false, true, L[0].ln1_g, L[0].ln1_b, nullptr);
    }
    // tree verify / draft levels: attention_tree.cu (one CTA per row tile and head)
    int tree_w = 0, n_ttiles = 0, tree_nodes = 0;
    if (f.tree && f.decode) {
        if (f.tree->size() > static_cast<size_t>(max_seqs_ + max_rows_))
            throw std::logic_error("forward: decode attention groups exceed capacity");
        h2d(d_tgroups_, f.tree->data(), f.tree->size(), st_);
    } else if (f.tree) {
        int mx = 1;
        for (const auto& g : *f.tree) {
            mx = std::max(mx, g.nrows);
            tree_nodes = std::max(tree_nodes, g.n_nodes);
        }
        tree_w = tree_attn_warps(mx, static_cast<int>(f.tree->size()), dims_.heads, d / H, tree_nodes);
        build_tree_tiles(*f.tree, tree_w, ttiles_);
        n_ttiles = static_cast<int>(ttiles_.size());
        if (f.tree->size() > static_cast<size_t>(max_seqs_ + max_rows_) ||
            ttiles_.size() > static_cast<size_t>(max_seqs_ + max_rows_))
            throw std::logic_error("forward: tree attention tables exceed capacity");
        h2d(d_tgroups_, f.tree->data(), f.tree->size(), st_);
        h2d(d_ttiles_, ttiles_.data(), ttiles_.size(), st_);
    }
    // rows sharing a committed prefix (tree verify, draft levels): shared tiles of <= 8 rows
    int n_tiles = 0, qw = 1;
    long long n_items = 0;
    if (!f.tree && f.groups && group_attn_enabled(static_cast<int>(f.groups->size()), M)) {
        qw = attn_tile_qw(*f.groups);
        n_items = build_attn_tiles(*f.groups, htiles_, qw, f.groups_exact);
        n_tiles = static_cast<int>(htiles_.size());
        if (n_tiles > 2 * max_rows_) throw std::logic_error("forward: attention tiles exceed capacity");
        h2d(tiles_, htiles_.data(), htiles_.size(), st_);
    }
    const size_t lstride = static_cast<size_t>(kv.n_slots) * d;
    const double attn_bytes = f.attn_kv_unique * d * 4.0 + row_bytes * 1.5;
    const double attn_flops = 4.0 * f.attn_row_keys * d;
    for (size_t l = 0; l < L.size(); ++l) {
        const LayerDev& W = L[l];
        GemmEpi eq;
        eq.kind = kEpiQKV;
        eq.f32 = q_;
        eq.kv_dst = rows_.kv_dst;
        eq.K = kv.K + l * lstride;
        eq.V = kv.V + l * lstride;
        eq.ld = 3 * d;
        eq.d = d;
        gemm(W.qkv, act_a_, M, eq, kClsGemm, 8.0 / 3.0);
        e0 = pbeg();
        if (f.tree && f.decode)
            launch_attention_decode(q_, f.draft ? dkmap_ : tkmap_, f.draft ? dvmap_ : tvmap_,
                                    static_cast<long long>(l) * kv.n_slots, eq.K, eq.V, d_tgroups_,
                                    static_cast<int>(f.tree->size()), f.decode_max_ctx, H, d, att_, st_);
        else if (f.tree)
            launch_attention_tree(q_, f.draft ? dkmap_ : tkmap_, f.draft ? dvmap_ : tvmap_,
                                  static_cast<long long>(l) * kv.n_slots, eq.K, eq.V, ar, d_tgroups_, d_ttiles_, n_ttiles,
                                  tree_w, H, d, tree_nodes, att_, st_);
        else if (n_tiles)
            launch_attention_tiles(q_, eq.K, eq.V, kv.n_slots, ar, M, tiles_, n_tiles, n_items, qw, H, d, f.max_vlen,
                                   asc_, att_, st_, f.merge_tiles);
        else
            launch_attention(q_, eq.K, eq.V, kv.n_slots, ar, M, H, d, f.max_vlen, f.attn_row_keys, asc_, att_, st_);
        pend(kClsAttn, e0, attn_bytes, attn_flops);
        count();
        gemm_resid_ln(W.wo, act_att_, M, true, false, W.ln2_g, W.ln2_b, nullptr);
        GemmEpi eg;
        eg.kind = kEpiGeluBF16;
        eg.b16 = h_;
        eg.ld = F;
        gemm(W.w1, act_a_, M, eg, kClsGemm, 2.0);
        const bool last = l + 1 == L.size();
        const float* g = last ? (f.draft ? dlnf_g_ : lnf_g_) : L[l + 1].ln1_g;
        const float* b = last ? (f.draft ? dlnf_b_ : lnf_b_) : L[l + 1].ln1_b;
        gemm_resid_ln(W.w2, act_h_, M, true, false, g, b, last ? f.y_out : nullptr);
    }
    if (f.logits) {
        if (f.lm_idx) {
            launch_gather_rows_bf16(a_, f.lm_idx, f.lm_rows, d, a2_, st_);
            count();
            lm_head(a2_, act_a2_, f.lm_rows, f.logits_out);
        } else {
            lm_head(a_, act_a_, M, f.logits_out);
        }
    }
}

// ------------------------------------------------------------------ profiler (CUDA events)
int Engine::pbeg() {
    if (!prof_) return -1;
    if (ev_used_ >= static_cast<int>(evs_.size())) {
        cudaEvent_t e;
        SGB_CUDA(cudaEventCreate(&e));
        evs_.push_back(e);
    }
    SGB_CUDA(cudaEventRecord(evs_[ev_used_], st_));
    return ev_used_++;
}

void Engine::pend(int cls, int e0, double bytes, double flops) {
    if (!prof_ || e0 < 0) return;
    const int e1 = pbeg();
    precs_.push_back(PRec{cls, e0, e1, bytes, flops});
}

void Engine::pflush() {
    if (precs_.empty()) {
        ev_used_ = 0;
        return;
    }
    SGB_CUDA(cudaStreamSynchronize(st_));
    for (const PRec& r : precs_) {
        float ms = 0.f;
        SGB_CUDA(cudaEventElapsedTime(&ms, evs_[r.e0], evs_[r.e1]));
        KernelProfile& k = prof_cls_[r.cls];
        k.ms += ms;
        k.launches += 1;
        k.bytes += r.bytes;
        k.flops += r.flops;
    }
    precs_.clear();
    ev_used_ = 0;
}

void Engine::set_profiling(bool on) {
    pflush();
    prof_ = on;
}

void Engine::read_profile(KernelProfile* out, int n, bool reset) {
    pflush();
    for (int i = 0; i < n && i < kNumCls; ++i) out[i] = prof_cls_[i];
    if (reset)
        for (auto& k : prof_cls_) k = KernelProfile{};
}

void Engine::upload_rows_host(int M, const std::vector<int>& tok, const std::vector<int>& pos,
                              const std::vector<long long>& kv_dst, const std::vector<long long>& ctx_base,
                              const std::vector<int>& ctx_len, const std::vector<int>& chain_len,
                              const std::vector<long long>& chain, const std::vector<long long>* feat_off) {
    if (!tok.empty()) h2d(rows_.tok, tok.data(), M, st_);
    h2d(rows_.pos, pos.data(), M, st_);
    h2d(rows_.kv_dst, kv_dst.data(), M, st_);
    h2d(rows_.ctx_base, ctx_base.data(), M, st_);
    h2d(rows_.ctx_len, ctx_len.data(), M, st_);
    h2d(rows_.chain_len, chain_len.data(), M, st_);
    if (!chain.empty()) h2d(rows_.chain, chain.data(), static_cast<size_t>(M) * kMaxChain, st_);
    if (feat_off) h2d(rows_.feat_off, feat_off->data(), M, st_);
}

// ------------------------------------------------------------------ C_peak calibration
double Engine::latency_probe(int b, int warmup, int reps) {
    if (b < 1 || b > max_rows_) throw std::invalid_argument("latency_probe: batch outside [1, max_rows]");
    if (b > tkv_.n_slots) throw std::invalid_argument("latency_probe: batch exceeds KV slots");
    if (!target_ready_) throw std::runtime_error("weights not uploaded");
    // rows of the reference latency_fn: token kEosToken at position 0, self-only mask ->
    // each row's only key is its own (written to a distinct KV slot)
    std::vector<int> tok(b, 1), pos(b, 0), cl(b, 0), chl(b, 1);
    std::vector<long long> kvd(b), cb(b, 0), ch(static_cast<size_t>(b) * kMaxChain, 0);
    for (int i = 0; i < b; ++i) {
        kvd[i] = i;
        ch[static_cast<size_t>(i) * kMaxChain] = i;
    }
    upload_rows_host(b, tok, pos, kvd, cb, cl, chl, ch, nullptr);
    Fwd f;
    f.M = b;
    f.y_out = y_;
    f.logits = true;
    f.logits_out = logits_;
    f.max_vlen = 1;
    f.attn_kv_unique = b;
    f.attn_row_keys = b;
    std::vector<double> t(reps);
    for (int w = 0; w < warmup; ++w) forward(f);
    for (int r = 0; r < reps; ++r) {
        SGB_CUDA(cudaEventRecord(ev0_, st_));
        forward(f);
        SGB_CUDA(cudaEventRecord(ev1_, st_));
        SGB_CUDA(cudaEventSynchronize(ev1_));
        float ms = 0.f;
        SGB_CUDA(cudaEventElapsedTime(&ms, ev0_, ev1_));
        t[r] = ms * 1e-3;
    }
    std::nth_element(t.begin(), t.begin() + reps / 2, t.end());
    return t[reps / 2];
}

// ------------------------------------------------------------------ per-op parity entry points
void Engine::cache_reset(int slot, bool draft) {
    if (slot < 0 || slot >= max_seqs_) throw std::invalid_argument("cache slot out of range");
    (draft ? cache_len_d_ : cache_len_t_)[slot] = 0;
}
int Engine::cache_len(int slot, bool draft) const {
    if (slot < 0 || slot >= max_seqs_) throw std::invalid_argument("cache slot out of range");
    return (draft ? cache_len_d_ : cache_len_t_)[slot];
}

void Engine::cache_read(int slot, bool draft, float* k, float* v) {
    const KvStore& kv = draft ? dkv_ : tkv_;
    const int len = cache_len(slot, draft), d = dims_.d;
    std::vector<__nv_bfloat16> tmp(static_cast<size_t>(len) * d);
    SGB_CUDA(cudaStreamSynchronize(st_));
    for (int l = 0; l < kv.layers; ++l) {
        for (int w = 0; w < 2; ++w) {
            const __nv_bfloat16* src = (w ? kv.V : kv.K) + (static_cast<size_t>(l) * kv.n_slots + slot * kv.seq_stride) * d;
            SGB_CUDA(cudaMemcpy(tmp.data(), src, tmp.size() * 2, cudaMemcpyDeviceToHost));
            float* dst = (w ? v : k) + static_cast<size_t>(l) * len * d;
            for (size_t i = 0; i < tmp.size(); ++i) dst[i] = __bfloat162float(tmp[i]);
        }
    }
}

void Engine::cache_gather_tail(int slot, int base, const int* keep, int n) {  // tinylm.hpp:254-268
    int& len = cache_len_t_.at(slot);
    if (base < 0 || base > len) throw std::invalid_argument("gather_tail: base beyond length");
    for (int i = 0; i < n; ++i) {
        if (keep[i] < 0 || base + keep[i] >= len || (i > 0 && keep[i] <= keep[i - 1]))
            throw std::invalid_argument("gather_tail: keep must be strictly increasing and in range");
    }
    const int d = dims_.d;
    for (int l = 0; l < tkv_.layers; ++l)
        for (int i = 0; i < n; ++i) {
            if (keep[i] == i) continue;
            for (int w = 0; w < 2; ++w) {
                __nv_bfloat16* P = (w ? tkv_.V : tkv_.K) + (static_cast<size_t>(l) * tkv_.n_slots + slot * tkv_.seq_stride) * d;
                SGB_CUDA(cudaMemcpyAsync(P + static_cast<size_t>(base + i) * d, P + static_cast<size_t>(base + keep[i]) * d,
                                         d * 2, cudaMemcpyDeviceToDevice, st_));
            }
        }
    len = base + n;
    SGB_CUDA(cudaStreamSynchronize(st_));
}

void Engine::forward_target(int slot, const int* tokens, const int* positions, int rows, const unsigned char* mask,
                            float* logits, float* hidden) {  // tinylm.hpp:422-463
    if (rows <= 0) throw std::invalid_argument("forward_target: empty input");
    for (int i = 0; i < rows; ++i) {
        if (tokens[i] < 0 || tokens[i] >= dims_.vocab)
            throw std::invalid_argument("forward_target: token id out of range");
        if (positions[i] < 0 || positions[i] >= dims_.max_seq)
            throw std::out_of_range("forward_target: position beyond max_seq_len");
    }
    int& len = cache_len_t_.at(slot);
    if (len + rows > dims_.max_seq) throw std::out_of_range("forward_target: cache capacity");
    const long long base = static_cast<long long>(slot) * tkv_.seq_stride;
    std::vector<int> tok(tokens, tokens + rows), pos(positions, positions + rows), cl(rows), chl(rows, 0);
    std::vector<long long> kvd(rows), cb(rows, base), ch(static_cast<size_t>(rows) * kMaxChain, 0);
    for (int i = 0; i < rows; ++i) {
        if (!mask) {
            kvd[i] = base + len + i;
            cl[i] = len + i + 1;
        } else {
            kvd[i] = tkv_.scratch_base + i;
            cl[i] = len;
            int c = 0;
            for (int j = 0; j < rows; ++j)
                if (mask[static_cast<size_t>(i) * rows + j]) {
                    if (c >= kMaxChain) throw std::invalid_argument("forward_target: mask row exceeds tree depth");
                    ch[static_cast<size_t>(i) * kMaxChain + c++] = tkv_.scratch_base + j;
                }
            chl[i] = c;
        }
    }
    upload_rows_host(rows, tok, pos, kvd, cb, cl, chl, ch, nullptr);
    Fwd f;
    f.M = rows;
    f.y_out = y_;
    f.logits = true;
    f.logits_out = logits_;
    f.max_vlen = len + rows;
    f.attn_kv_unique = len + rows;
    f.attn_row_keys = static_cast<double>(rows) * (len + rows);
    forward(f);
    if (mask) {  // extend the cache by every forwarded row (tinylm.hpp:405-412)
        const int d = dims_.d;
        for (int l = 0; l < tkv_.layers; ++l)
            for (int w = 0; w < 2; ++w) {
                __nv_bfloat16* P = (w ? tkv_.V : tkv_.K) + static_cast<size_t>(l) * tkv_.n_slots * d;
                SGB_CUDA(cudaMemcpyAsync(P + (base + len) * d, P + tkv_.scratch_base * d,
                                         static_cast<size_t>(rows) * d * 2, cudaMemcpyDeviceToDevice, st_));
            }
    }
    len += rows;
    if (logits) d2h(logits, logits_, static_cast<size_t>(rows) * dims_.vocab, st_);
    if (hidden) d2h(hidden, y_, static_cast<size_t>(rows) * dims_.d, st_);
    SGB_CUDA(cudaStreamSynchronize(st_));
}

void Engine::forward_draft(int slot, const int* tokens, const float* prev_feat, const int* positions, int rows,
                           bool extend, float* feats, float* logits) {  // tinylm.hpp:502-563
    if (rows <= 0) throw std::invalid_argument("forward_draft: empty input");
    for (int i = 0; i < rows; ++i) {
        if (tokens[i] < 0 || tokens[i] >= dims_.vocab)
            throw std::invalid_argument("forward_draft: token id out of range");
        if (positions[i] < 0 || positions[i] >= dims_.max_seq)
            throw std::out_of_range("forward_draft: position beyond max_seq_len");
    }
    int& len = cache_len_d_.at(slot);
    if (len + rows > dims_.max_seq) throw std::out_of_range("forward_draft: cache capacity");
    if (!extend && rows > kMaxChain) throw std::invalid_argument("forward_draft: read-only rows exceed chain");
    const long long base = static_cast<long long>(slot) * dkv_.seq_stride;
    std::vector<int> tok(tokens, tokens + rows), pos(positions, positions + rows), cl(rows), chl(rows, 0);
    std::vector<long long> kvd(rows), cb(rows, base), ch(static_cast<size_t>(rows) * kMaxChain, 0), fo(rows);
    for (int i = 0; i < rows; ++i) {
        fo[i] = static_cast<long long>(i) * dims_.d;
        if (extend) {
            kvd[i] = base + len + i;
            cl[i] = len + i + 1;
        } else {
            kvd[i] = dkv_.scratch_base + i;
            cl[i] = len;
            for (int j = 0; j <= i; ++j) ch[static_cast<size_t>(i) * kMaxChain + j] = dkv_.scratch_base + j;
            chl[i] = i + 1;
        }
    }
    upload_rows_host(rows, tok, pos, kvd, cb, cl, chl, ch, &fo);
    h2d(featin_, prev_feat, static_cast<size_t>(rows) * dims_.d, st_);
    Fwd f;
    f.M = rows;
    f.draft = true;
    f.feat_base = featin_;
    f.y_out = y_;
    f.logits = true;
    f.logits_out = logits_;
    f.max_vlen = len + rows;
    f.attn_kv_unique = len + rows;
    f.attn_row_keys = static_cast<double>(rows) * (len + rows);
    forward(f);
    if (extend) len += rows;
    if (logits) d2h(logits, logits_, static_cast<size_t>(rows) * dims_.vocab, st_);
    if (feats) d2h(feats, y_, static_cast<size_t>(rows) * dims_.d, st_);
    SGB_CUDA(cudaStreamSynchronize(st_));
}

void Engine::emit(const float* logits, int rows, int vocab, double temperature, const unsigned long long* seeds,
                  const int* key_pos, int* out, const double* uniforms, int* exact_rows) {
    if (vocab != dims_.vocab) throw std::invalid_argument("emit: vocab mismatch");
    if (rows <= 0 || rows > max_rows_) throw std::invalid_argument("emit: bad row count");
    if (temperature < 0) throw std::invalid_argument("sample_token: negative temperature");
    h2d(logits_, logits, static_cast<size_t>(rows) * vocab, st_);
    double* du = nullptr;
    if (uniforms) {
        for (int i = 0; i < rows; ++i)
            if (!(uniforms[i] >= 0.0 && uniforms[i] < 1.0)) throw std::invalid_argument("sample: uniform outside [0, 1)");
        du = reinterpret_cast<double*>(misc_l_);  // 2R + 2S words
        h2d(du, uniforms, rows, st_);
    } else {
        h2d(rows_.seed, seeds, rows, st_);
        h2d(rows_.key_pos, key_pos, rows, st_);
    }
    SGB_CUDA(cudaMemsetAsync(err_, 0, sizeof(int), st_));
    launch_emit(logits_, vocab, nullptr, rows_.seed, rows_.key_pos, rows, temperature, emitted_, err_, rsc_, st_, du);
    d2h(out, emitted_, rows, st_);
    if (exact_rows) {
        if (temperature > 0) d2h(exact_rows, rsc_.exact, rows, st_);
        else std::fill(exact_rows, exact_rows + rows, 0);
    }
    int err = 0;
    d2h(&err, err_, 1, st_);
    SGB_CUDA(cudaStreamSynchronize(st_));
    if (err & 2) throw std::domain_error("sample_token: NaN logit");
    if (err & 4) throw std::domain_error("sample_token: all logits are -inf");
}

void Engine::debug_exp(const double* x, size_t n, double* y) {
    double* dx = dalloc<double>(n);
    double* dy = dalloc<double>(n);
    h2d(dx, x, n, st_);
    launch_debug_exp(dx, n, dy, st_);
    d2h(y, dy, n, st_);
    SGB_CUDA(cudaStreamSynchronize(st_));
    cudaFree(dx);
    cudaFree(dy);
}

unsigned long long Engine::exact_draws() {
    unsigned long long n = 0;
    SGB_CUDA(cudaMemcpyAsync(&n, rsc_.n_exact, sizeof(n), cudaMemcpyDeviceToHost, st_));
    SGB_CUDA(cudaStreamSynchronize(st_));
    return n;
}

void Engine::topk_logsoftmax(const float* logits, int rows, int vocab, int k, int* tok, double* lp) {
    if (vocab != dims_.vocab) throw std::invalid_argument("topk: vocab mismatch");
    if (rows <= 0 || rows > max_rows_) throw std::invalid_argument("topk: bad row count");
    k = std::min(k, vocab);
    h2d(logits_, logits, static_cast<size_t>(rows) * vocab, st_);
    launch_topk_lsm(logits_, vocab, rows, k, topk_tok_, topk_lp_, rsc_, st_);
    d2h(tok, topk_tok_, static_cast<size_t>(rows) * k, st_);
    d2h(lp, topk_lp_, static_cast<size_t>(rows) * k, st_);
    SGB_CUDA(cudaStreamSynchronize(st_));
}

Engine::DebugTree Engine::debug_tree_cb(int root_token, int k, int l, int n_verify,
                                        void (*fn)(void*, int, const int*, const int*, const int*, int, float*),
                                        void* ctx) {
    const int V = dims_.vocab;
    if (k < 0 || l < 0) throw std::invalid_argument("expand_tree: negative k_draft or l_draft");
    if (n_verify < 1) throw std::invalid_argument("rerank_candidates: n_verify must be >= 1");
    if (k > k_max_ || l > l_max_) throw std::invalid_argument("debug_tree: k/l beyond engine capacity");
    const int ke = (k == 0 || l == 0) ? 0 : std::min(k, V);
    const int le = ke == 0 ? 0 : l;
    const int nodes = ke ? tree_cap(ke, le) : 1;
    StepSeqDev sd{0, 0, ke, le, std::min(n_verify, nodes), 0, ke ? 0 : -1, dims_.max_seq};
    h2d(ss_.tokens, &root_token, 1, st_);
    h2d(steps_, &sd, 1, st_);
    std::vector<float> lg(static_cast<size_t>(std::max(1, ke)) * V);
    if (ke) {
        int id0 = 0, t0 = root_token, p0 = -1;
        fn(ctx, 1, &id0, &t0, &p0, 1, lg.data());
        h2d(logits_, lg.data(), V, st_);
        launch_topk_lsm(logits_, V, 1, ke, topk_tok_, topk_lp_, rsc_, st_);
    }
    launch_tree_root(1, steps_, ss_, tr_, topk_tok_, topk_lp_, std::max(1, ke), st_);
    const int zero = 0;
    h2d(drow_, &zero, 1, st_);
    for (int level = 2; level <= le; ++level) {
        launch_tree_frontier(1, level, steps_, drow_, ss_, tr_, rows_, dkv_.seq_stride, dkv_.scratch_base, dims_.d,
                             st_);
        int n = 0;
        d2h(&n, tr_.n_nodes, 1, st_);
        SGB_CUDA(cudaStreamSynchronize(st_));
        std::vector<int> fr(ke), tok(n), par(n);
        d2h(fr.data(), tr_.frontier, ke, st_);
        d2h(tok.data(), tr_.tok, n, st_);
        d2h(par.data(), tr_.par, n, st_);
        SGB_CUDA(cudaStreamSynchronize(st_));
        fn(ctx, ke, fr.data(), tok.data(), par.data(), n, lg.data());
        h2d(logits_, lg.data(), static_cast<size_t>(ke) * V, st_);
        launch_topk_lsm(logits_, V, ke, ke, topk_tok_, topk_lp_, rsc_, st_);
        launch_tree_expand(1, level, steps_, drow_, tr_, topk_tok_, topk_lp_, st_);
    }
    SGB_CUDA(cudaMemsetAsync(mask_dbg_, 0, static_cast<size_t>(sd.nsel) * sd.nsel, st_));
    SGB_CUDA(cudaMemsetAsync(err_, 0, sizeof(int), st_));
    launch_tree_select(1, steps_, ss_, tr_, rows_, tkv_.seq_stride, tkv_.scratch_base, mask_dbg_, err_, st_);
    DebugTree out;
    int n = 0;
    d2h(&n, tr_.n_nodes, 1, st_);
    SGB_CUDA(cudaStreamSynchronize(st_));
    out.tok.resize(n);
    out.par.resize(n);
    out.dep.resize(n);
    out.lp.resize(n);
    out.conf.resize(n);
    out.sel.resize(sd.nsel);
    out.mask.resize(static_cast<size_t>(sd.nsel) * sd.nsel);
    d2h(out.tok.data(), tr_.tok, n, st_);
    d2h(out.par.data(), tr_.par, n, st_);
    d2h(out.dep.data(), tr_.dep, n, st_);
    d2h(out.lp.data(), tr_.lp, n, st_);
    d2h(out.conf.data(), tr_.conf, n, st_);
    d2h(out.sel.data(), tr_.sel, sd.nsel, st_);
    d2h(out.mask.data(), mask_dbg_, out.mask.size(), st_);
    int err = 0;
    d2h(&err, err_, 1, st_);
    SGB_CUDA(cudaStreamSynchronize(st_));
    if (err & 8) throw std::invalid_argument("build_tree_mask: closure violation");
    return out;
}

void Engine::reject_alloc() {
    if (qbuf_) return;
    const size_t R = max_rows_, V = dims_.vocab, S = max_seqs_;
    qbuf_ = dalloc<float>(R * V);
    qstat_ = dalloc<double>(2 * R);
    rkeys_ = dalloc<unsigned long long>(R);
    tr_.qrow = dalloc<int>(S * static_cast<size_t>(tr_.tmax));
}

// ------------------------------------------------------------------ the rollout
RolloutResult Engine::rollout(const RolloutArgs& a) {
    NvtxRange nv_rollout("sgb rollout");
    const ModelDims& mc = dims_;
    const int d = mc.d, V = mc.vocab, T = mc.max_seq;
    // validation (scheduler.cpp:240-249)
    if (a.prompts.empty()) throw std::invalid_argument("generate: prompts must be non-empty");
    if (a.g < 1) throw std::invalid_argument("generate: g must be >= 1");
    if (a.c_peak < 1) throw std::invalid_argument("generate: c_peak must be >= 1");
    for (const auto& pr : a.prompts) {
        if (pr.empty()) throw std::invalid_argument("generate: zero-length prompt");
        if (static_cast<int>(pr.size()) > T - 1)
            throw std::invalid_argument("generate: prompt longer than max_seq_len - 1");
        for (int t : pr)
            if (t < 0 || t >= V) throw std::invalid_argument("forward_target: token id out of range");
    }
    if (a.mode == 1) validate_spec(a.fixed, a.alpha, a.k_max, a.l_max, a.c_peak);
    if (a.k_max > k_max_ || a.l_max > l_max_)
        throw std::invalid_argument("generate: k_max/l_max exceed the engine's tree capacity");
    if (a.temperature < 0) throw std::invalid_argument("sample_token: negative temperature");
    if (a.acceptance < 0 || a.acceptance > 1) throw std::invalid_argument("generate: unknown acceptance mode");
    if (!target_ready_ || !draft_ready_) throw std::runtime_error("weights not uploaded");
    const bool rej = a.acceptance == 1 && a.temperature > 0;  // at T = 0 both modes are greedy strict match
    if (rej) reject_alloc();
    tr_.static_rank = rej ? 1 : 0;
    const int P = static_cast<int>(a.prompts.size());
    const int n_seqs = P * a.g;
    const int G = a.g;
    if (G > max_seqs_) throw std::invalid_argument("generate: group size exceeds engine max_seqs");
    if (G > max_rows_) throw std::invalid_argument("generate: group size exceeds engine max_rows");
    if (!a.seq_max_new.empty() && static_cast<int>(a.seq_max_new.size()) != n_seqs)
        throw std::invalid_argument("generate: seq_max_new size mismatch");

    RolloutResult res;
    const long long launches0 = launches_;
    SGB_CUDA(cudaMemsetAsync(err_, 0, sizeof(int), st_));

    // ---------------- sequences, KV regions and admission
    // The reference admits every sequence at once with its own KvCache (scheduler.cpp:259-294).
    // Here the KV store holds max_seqs_ sequence REGIONS (one region = max_seq_len slots of every
    // layer), handed out in aligned blocks of G to whole query groups (the members read their
    // prompt K/V from the group leader's region). When a rollout has more sequences than
    // regions it runs in waves: a group's regions are recycled once all its members finished
    // (their tokens and features copied out first) and the next pending group is admitted and
    // prefilled at that step boundary. Sequence ids, seeds and caps stay global (sid order).
    const int S = max_seqs_;
    const int n_gslots = S / G;
    std::vector<int> sid_of(S, -1), len(S, 0), len_cap(S, 0), fin(S, 1), dft_len(S, 0), plen(S, 0);
    std::vector<unsigned long long> seeds(S, 0);
    std::vector<int> sid_cap(n_seqs), sid_len(n_seqs, 0), sid_eos(n_seqs, 0);
    std::vector<unsigned long long> sid_seed(n_seqs);
    for (int sid = 0; sid < n_seqs; ++sid) {
        const int q = static_cast<int>(a.prompts[sid / G].size());
        sid_seed[sid] = mix_key_host(a.seed, static_cast<uint64_t>(sid + a.sid_offset) + 1);
        const int mn = a.seq_max_new.empty() ? a.max_new_tokens : a.seq_max_new[sid];
        sid_cap[sid] = mn > 0 ? std::min(T, q + mn) : T;
    }
    res.tokens.resize(n_seqs);
    res.prompt_len.resize(n_seqs);
    res.hit_eos.assign(n_seqs, 0);
    if (a.want_features && !a.features_out) res.features.resize(n_seqs);
    std::vector<int> gslot_group(n_gslots, -1);  // query group held by a block of G regions
    int next_group = 0;
    bool waves = false;
    for (const auto& pr : a.prompts) res.h2d_bytes += static_cast<long long>(pr.size()) * sizeof(int);
    SGB_CUDA(cudaEventRecord(ev0_, st_));  // inputs resident in HBM from here on

    // copy a retired sequence's tokens (+ features) to the host result (scheduler.cpp:343-353)
    auto retire = [&](int slot) {
        const int sid = sid_of[slot];
        auto& tk = res.tokens[sid];
        tk.resize(len[slot]);
        d2h(tk.data(), ss_.tokens + static_cast<size_t>(slot) * T, len[slot], st_);
        if (a.want_features) {
            const size_t nf = static_cast<size_t>(len[slot] - 1) * d;
            float* dst = a.features_out ? a.features_out + static_cast<size_t>(sid) * (T - 1) * d
                                        : (res.features[sid].resize(nf), res.features[sid].data());
            d2h(dst, feats_ + static_cast<size_t>(slot) * T * d, nf, st_);
        }
        d2h(&sid_eos[sid], ss_.hit_eos + slot, 1, st_);
        sid_len[sid] = len[slot];
        sid_of[slot] = -1;
    };

    // ---------------- prefill of newly admitted groups: one forward per chunk of distinct
    // prompts (scheduler.cpp:259-294); the prompt K/V is copied to the G members
    auto prefill = [&](const std::vector<std::pair<int, int>>& adm) {  // (query group, gslot)
        const int NA = static_cast<int>(adm.size());
        int ai = 0;
        while (ai < NA) {
            // a chunk is bounded by its prompt rows AND by its np * g first-token emissions (both
            // index row-sized buffers: lm_idx_, rows_.seed, the sampling scratch)
            int rows = 0, ae = ai;
            while (ae < NA && rows + static_cast<int>(a.prompts[adm[ae].first].size()) <= max_rows_ &&
                   (ae - ai + 1) * G <= max_rows_)
                rows += a.prompts[adm[ae++].first].size();
            if (ae == ai) throw std::invalid_argument("generate: prompt longer than engine max_rows");
            std::vector<int> tok, pos, cl, chl, last_rows;
            std::vector<long long> kvd, cb;
            int maxq = 0;
            for (int x = ai; x < ae; ++x) {
                const int p2 = adm[x].first, s0 = adm[x].second * G;
                const int q = static_cast<int>(a.prompts[p2].size());
                maxq = std::max(maxq, q);
                for (int t = 0; t < q; ++t) {
                    tok.push_back(a.prompts[p2][t]);
                    pos.push_back(t);
                    kvd.push_back(static_cast<long long>(s0) * T + t);
                    cb.push_back(static_cast<long long>(s0) * T);
                    cl.push_back(t + 1);
                    chl.push_back(0);
                }
                last_rows.push_back(static_cast<int>(tok.size()) - 1);
            }
            upload_rows_host(rows, tok, pos, kvd, cb, cl, chl, {}, nullptr);
            const int np = ae - ai;
            h2d(lm_idx_, last_rows.data(), np, st_);
            Fwd f;
            f.M = rows;
            f.y_out = y_;
            f.logits = true;
            f.lm_rows = np;
            f.lm_idx = lm_idx_;
            f.logits_out = logits_;
            f.max_vlen = maxq;
            f.attn_kv_unique = rows;
            for (int x = ai; x < ae; ++x) {
                const double q = static_cast<double>(a.prompts[adm[x].first].size());
                f.attn_row_keys += q * (q + 1) / 2;
            }
            forward(f);
            res.target_forwards++;
            // features of every member: feats[s][t] = hidden[row]
            std::vector<int> src_row;
            std::vector<long long> dst_off;
            std::vector<int> srcs, dsts, pl, emseq, emq, emcap, emrow, emkey;
            std::vector<unsigned long long> emseed;
            int row0 = 0;
            for (int x = ai; x < ae; ++x) {
                const int p2 = adm[x].first, s0 = adm[x].second * G;
                const int q = static_cast<int>(a.prompts[p2].size());
                for (int r = 0; r < G; ++r) {
                    const int s = s0 + r;
                    for (int t = 0; t < q; ++t) {
                        src_row.push_back(row0 + t);
                        dst_off.push_back((static_cast<long long>(s) * T + t) * d);
                    }
                    if (r > 0) {
                        srcs.push_back(s0);
                        dsts.push_back(s);
                        pl.push_back(q);
                    }
                    emseq.push_back(s);
                    emq.push_back(q);
                    emcap.push_back(len_cap[s]);
                    emrow.push_back(x - ai);
                    emseed.push_back(seeds[s]);
                    emkey.push_back(q);
                }
                row0 += q;
            }
            const int nr = static_cast<int>(src_row.size());
            for (int off = 0; off < nr; off += max_rows_) {  // chunk the copy descriptors
                const int c = std::min(max_rows_, nr - off);
                h2d(misc_i_, src_row.data() + off, c, st_);
                h2d(misc_l_, dst_off.data() + off, c, st_);
                launch_copy_rows_f32(y_, misc_i_, misc_l_, c, d, feats_, st_);
                count();
                SGB_CUDA(cudaStreamSynchronize(st_));
            }
            if (!srcs.empty()) {
                const int n = static_cast<int>(srcs.size());
                int* b = misc_i_;
                h2d(b, srcs.data(), n, st_);
                h2d(b + n, dsts.data(), n, st_);
                h2d(b + 2 * n, pl.data(), n, st_);
                launch_copy_kv_prefix(b, b + n, b + 2 * n, n, maxq, tkv_.layers, d, tkv_.K, tkv_.V, tkv_.n_slots * d,
                                      tkv_.seq_stride, st_);
                count();
                SGB_CUDA(cudaStreamSynchronize(st_));
            }
            const int ne = static_cast<int>(emseq.size());
            int* b = misc_i_;
            h2d(b, emrow.data(), ne, st_);
            h2d(b + ne, emkey.data(), ne, st_);
            h2d(rows_.seed, emseed.data(), ne, st_);
            launch_emit(logits_, V, b, rows_.seed, b + ne, ne, a.temperature, emitted_, err_, rsc_, st_);
            count(emit_launches(a.temperature) - 1);
            h2d(b + 2 * ne, emseq.data(), ne, st_);
            h2d(b + 3 * ne, emq.data(), ne, st_);
            h2d(lm_idx_, emcap.data(), ne, st_);
            launch_prefill_commit(ne, b + 2 * ne, b + 3 * ne, lm_idx_, emitted_, ss_, st_);
            count(2);
            SGB_CUDA(cudaStreamSynchronize(st_));
            ai = ae;
        }
        std::vector<int> t1(S), f1(S);
        d2h(t1.data(), ss_.len, S, st_);
        d2h(f1.data(), ss_.finished, S, st_);
        SGB_CUDA(cudaStreamSynchronize(st_));
        for (const auto& g2 : adm)
            for (int r = 0; r < G; ++r) {
                const int s = g2.second * G + r;
                len[s] = t1[s];
                fin[s] = f1[s];
            }
    };

    // admit pending query groups into free region blocks, then prefill them
    auto admit = [&]() {
        NvtxRange nv_admit("sgb admit + prefill");
        std::vector<std::pair<int, int>> adm;
        for (int gs = 0; gs < n_gslots && next_group < P; ++gs) {
            if (gslot_group[gs] >= 0) continue;
            const int pi = next_group++;
            gslot_group[gs] = pi;
            const int q = static_cast<int>(a.prompts[pi].size());
            for (int r = 0; r < G; ++r) {
                const int s = gs * G + r, sid = pi * G + r;
                sid_of[s] = sid;
                plen[s] = q;
                seeds[s] = sid_seed[sid];
                len_cap[s] = sid_cap[sid];
                dft_len[s] = 0;
                fin[s] = 0;
                res.prompt_len[sid] = q;
                h2d(ss_.tokens + static_cast<size_t>(s) * T, a.prompts[pi].data(), q, st_);
            }
            h2d(ss_.seed + gs * G, seeds.data() + gs * G, G, st_);
            adm.emplace_back(pi, gs);
        }
        if (!adm.empty()) prefill(adm);
    };
    admit();
    if (next_group < P) waves = true;

    // ---------------- step loop (scheduler.cpp:299-341)
    SGB_CUDA(cudaEventRecord(evs_a_, st_));  // prefill done; each step's end is timed against the last
    {
        float ms = 0.f;
        SGB_CUDA(cudaEventSynchronize(evs_a_));
        SGB_CUDA(cudaEventElapsedTime(&ms, ev0_, evs_a_));
        res.prefill_seconds = ms * 1e-3;
    }
    std::vector<StepSeqDev> hs;
    std::vector<int> drow, live;
    for (int step = 0;; ++step) {
        live.clear();
        for (int s = 0; s < S; ++s)
            if (sid_of[s] >= 0 && !fin[s]) live.push_back(s);
        const int B = static_cast<int>(live.size());
        if (B == 0) break;  // (pending groups are admitted at the end of the step that frees regions)
        const auto t_host0 = std::chrono::steady_clock::now();
        NvtxRange nv_step("sgb step");
        const int eff_b = a.early_term ? B : n_seqs;
        SpecCfg cfg;
        if (a.mode == 0) cfg = SpecCfg{1, 0, 0};
        else if (a.mode == 1) cfg = a.fixed;
        else cfg = plan(a.c_peak, eff_b, a.alpha, a.k_max, a.l_max);

        // per-sequence shapes (scheduler.cpp:125-133)
        hs.assign(B, StepSeqDev{});
        int vrows = 0, n_spec = 0, max_l = 0, max_p = 0, kstep = 0;
        for (int i = 0; i < B; ++i) {
            const int s = live[i];
            const int p = len[s] - 1;
            int l_eff = std::min(cfg.l_draft, len_cap[s] - 1 - p);
            int k_eff = l_eff >= 1 ? std::min(cfg.k_draft, V) : 0;
            if (k_eff == 0) l_eff = 0;
            const int nodes = k_eff ? tree_cap(k_eff, l_eff) : 1;
            StepSeqDev& e = hs[i];
            e.seq = s;
            e.p = p;
            e.k = k_eff;
            e.l = l_eff;
            e.nsel = std::min(cfg.n_verify, nodes);
            e.vrow_off = vrows;
            e.root_row = k_eff ? n_spec++ : -1;
            e.len_cap = len_cap[s];
            e.pre_len = plen[s];
            e.pre_base = static_cast<long long>(s - s % a.g) * tkv_.seq_stride;  // group leader's prompt K/V
            vrows += e.nsel;
            max_l = std::max(max_l, l_eff);
            max_p = std::max(max_p, p);
            if (k_eff) kstep = k_eff;
        }
        if (vrows > max_rows_) throw std::invalid_argument("generate: verify rows exceed engine max_rows");
        SGB_CUDA(cudaEventRecord(evs_c_, st_));  // the step's first device operation
        h2d(steps_, hs.data(), B, st_);
        StepStat stat;
        stat.b_cur = B;
        stat.n_verify = cfg.n_verify;
        stat.k_draft = cfg.k_draft;
        stat.l_draft = cfg.l_draft;
        stat.rows = vrows;

        std::optional<NvtxRange> nv_phase(std::in_place, n_spec > 0 ? "sgb draft" : "sgb plan");
        if (n_spec > 0) {
            // ---- draft catch-up over committed pairs (t_j, f_{j-1}), j = dft_len+1..p (scheduler.cpp:137-157)
            struct CU {
                int s, j, spec;
            };
            std::vector<CU> cu;
            for (int i = 0; i < B; ++i)
                if (hs[i].k) {
                    const int s = hs[i].seq;
                    for (int j = dft_len[s] + 1; j <= hs[i].p; ++j) cu.push_back({s, j, hs[i].root_row});
                }
            const int ncu = static_cast<int>(cu.size());
            for (int off = 0; off < ncu; off += max_rows_) {
                const int M = std::min(max_rows_, ncu - off);
                std::vector<int> seq(M), pos(M), cl(M), chl(M, 0), lastr, lasts;
                std::vector<long long> kvd(M), cb(M), fo(M), dsto;
                int maxj = 0;
                for (int r = 0; r < M; ++r) {
                    const CU& c = cu[off + r];
                    seq[r] = c.s;
                    pos[r] = c.j;
                    kvd[r] = static_cast<long long>(c.s) * T + (c.j - 1);
                    cb[r] = static_cast<long long>(c.s) * T;
                    cl[r] = c.j;
                    fo[r] = (static_cast<long long>(c.s) * T + (c.j - 1)) * d;
                    maxj = std::max(maxj, c.j);
                    const bool last = (off + r + 1 == ncu) || cu[off + r + 1].s != c.s;
                    if (last) {
                        lastr.push_back(r);
                        lasts.push_back(c.spec);
                        dsto.push_back((static_cast<long long>(c.s) * tr_.ds + 0) * d);
                    }
                }
                upload_rows_host(M, {}, pos, kvd, cb, cl, chl, {}, &fo);
                h2d(misc_i_, seq.data(), M, st_);
                launch_gather_tokens(misc_i_, rows_.pos, M, ss_, rows_.tok, st_);
                count();
                Fwd f;
                f.M = M;
                f.draft = true;
                f.feat_base = feats_;
                f.y_out = y_;
                f.max_vlen = maxj;
                for (int r = 0; r < M; ++r) f.attn_row_keys += pos[r];
                for (size_t t = 0; t < lastr.size(); ++t) f.attn_kv_unique += pos[lastr[t]];
                // a sequence's catch-up rows are consecutive pairs (causal): they share the keys
                // below their first row's, so those blocks run as shared tiles (attention.cu
                // prompt-style groups; each row's own tail per row -- identical bits)
                groups_.clear();
                for (int r = 0; r < M;) {
                    int e = r + 1;
                    while (e < M && seq[e] == seq[r]) ++e;
                    groups_.push_back({r, e - r, cl[r], cl[e - 1]});
                    r = e;
                }
                if (static_cast<int>(groups_.size()) < M) {
                    f.groups = &groups_;
                    f.groups_exact = false;
                    f.merge_tiles = true;
                }
                forward(f);
                res.draft_forwards++;
                stat.draft_rows += M;
                const int nl = static_cast<int>(lastr.size());
                if (nl) {
                    h2d(lm_idx_, lastr.data(), nl, st_);
                    h2d(misc_l_, dsto.data(), nl, st_);
                    launch_copy_rows_f32(y_, lm_idx_, misc_l_, nl, d, dfeat_, st_);  // root features
                    launch_gather_rows_bf16(a_, lm_idx_, nl, d, a2_ + static_cast<size_t>(lasts[0]) * d, st_);
                    count(2);
                }
                // no host sync: the next chunk's uploads and launches are stream-ordered after this one
            }
            for (int i = 0; i < B; ++i)
                if (hs[i].k) dft_len[hs[i].seq] = hs[i].p;
            // root logits -> level 1 (top-k children; rejection mode: k children sampled from q)
            int qoff = 0;
            if (rej) {
                std::vector<unsigned long long> keys(n_spec);
                for (int i = 0; i < B; ++i)
                    if (hs[i].k)
                        keys[hs[i].root_row] =
                            mix_key_host(mix_key_host(seeds[hs[i].seq], static_cast<uint64_t>(hs[i].p + 1)), 0xD5A0u);
                h2d(rkeys_, keys.data(), n_spec, st_);
                lm_head(a2_, act_a2_, n_spec, qbuf_);
                launch_sample_children(qbuf_, n_spec, V, kstep, a.temperature, rkeys_, topk_tok_, topk_lp_, qstat_, st_);
                qoff = n_spec;
            } else {
                lm_head(a2_, act_a2_, n_spec, logits_);
                launch_topk_lsm(logits_, V, n_spec, kstep, topk_tok_, topk_lp_, rsc_, st_);
            }
            launch_tree_root(B, steps_, ss_, tr_, topk_tok_, topk_lp_, kstep, st_);
            count(2);
            // levels 2..L: one batched draft forward per level
            if (max_l >= 2) {
                drow.assign(static_cast<size_t>(max_l - 1) * B, -1);
                std::vector<int> lvl_rows(max_l + 1, 0);
                for (int level = 2; level <= max_l; ++level) {
                    int r = 0;
                    for (int i = 0; i < B; ++i)
                        if (hs[i].k && hs[i].l >= level) {
                            drow[static_cast<size_t>(level - 2) * B + i] = r;
                            r += hs[i].k;
                        }
                    lvl_rows[level] = r;
                }
                h2d(drow_, drow.data(), drow.size(), st_);
                for (int level = 2; level <= max_l; ++level) {
                    const int R = lvl_rows[level];
                    if (R == 0) break;
                    if (R > max_rows_) throw std::invalid_argument("generate: draft rows exceed engine max_rows");
                    const int* dro = drow_ + static_cast<size_t>(level - 2) * B;
                    if (rej && qoff + R > max_rows_) throw std::invalid_argument("generate: draft q rows exceed max_rows");
                    launch_tree_frontier(B, level, steps_, dro, ss_, tr_, rows_, dkv_.seq_stride, dkv_.scratch_base,
                                         d, st_, rej ? qoff : -1);
                    count();
                    Fwd f;
                    f.M = R;
                    f.draft = true;
                    f.feat_base = dfeat_;
                    f.y_out = y_;
                    f.logits = true;
                    f.logits_out = rej ? qbuf_ + static_cast<size_t>(qoff) * V : logits_;
                    f.max_vlen = max_p + level;
                    groups_.clear();
                    tgroups_.clear();
                    for (int i = 0; i < B; ++i)
                        if (hs[i].k && hs[i].l >= level) {
                            f.attn_kv_unique += hs[i].p + level - 1;
                            f.attn_row_keys += static_cast<double>(hs[i].k) * (hs[i].p + level - 1);
                            const int r0 = drow[static_cast<size_t>(level - 2) * B + i];
                            groups_.push_back({r0, hs[i].k, hs[i].p, hs[i].p + level});
                            const int s = hs[i].seq;
                            // frontier rows: draft prefix (p keys), paths in the sequence's draft scratch
                            tgroups_.push_back(TreeGroupDev{r0, hs[i].k, hs[i].p, tr_.ds,
                                                            dkv_.scratch_base + static_cast<long long>(s) * tr_.ds,
                                                            static_cast<long long>(s) * dkv_.seq_stride,
                                                            static_cast<long long>(s) * dkv_.seq_stride, 0, 0});
                        }
                    f.groups = &groups_;
                    f.groups_exact = boundary_tiles();
                    f.merge_tiles = true;
                    static const int lvl_min = [] {
                        const char* v = getenv("SGB_TREE_LEVEL_MIN");  // A/B switch
                        return v ? atoi(v) : 3;
                    }();
                    if (kstep >= lvl_min && tree_attn_ok(tr_.ds)) f.tree = &tgroups_;
                    forward(f);
                    res.draft_forwards++;
                    stat.draft_rows += R;
                    launch_copy_rows_f32(y_, nullptr, rows_.out_off, R, d, dfeat_, st_);
                    if (rej) {
                        std::vector<unsigned long long> keys(R);
                        for (int i = 0; i < B; ++i) {
                            const int r0 = drow[static_cast<size_t>(level - 2) * B + i];
                            if (r0 < 0) continue;
                            for (int j = 0; j < hs[i].k; ++j)  // frontier node j's children sit at p + level
                                keys[r0 + j] = mix_key_host(
                                    mix_key_host(seeds[hs[i].seq], static_cast<uint64_t>(hs[i].p + level)), 0xD5A0u + j);
                        }
                        h2d(rkeys_, keys.data(), R, st_);
                        launch_sample_children(qbuf_ + static_cast<size_t>(qoff) * V, R, V, kstep, a.temperature, rkeys_,
                                               topk_tok_, topk_lp_, qstat_ + 2 * static_cast<size_t>(qoff), st_);
                        qoff += R;
                    } else {
                        launch_topk_lsm(logits_, V, R, kstep, topk_tok_, topk_lp_, rsc_, st_);
                    }
                    launch_tree_expand(B, level, steps_, dro, tr_, topk_tok_, topk_lp_, st_);
                    count(3);
                }
            }
        } else {
            launch_tree_root(B, steps_, ss_, tr_, topk_tok_, topk_lp_, 1, st_);
            count();
        }

        // ---- rerank + mask -> verify rows; one batched target forward (scheduler.cpp:208-217)
        nv_phase.reset();
        nv_phase.emplace("sgb verify");
        int pe0 = pbeg();
        launch_tree_select(B, steps_, ss_, tr_, rows_, tkv_.seq_stride, tkv_.scratch_base, nullptr, err_, st_);
        pend(kClsTree, pe0, 0, 0);
        count();
        Fwd f;
        f.M = vrows;
        f.prefix_share = a.g > 1;
        f.y_out = y_;
        f.logits = true;
        f.logits_out = logits_;
        f.max_vlen = max_p + max_l + 1;
        groups_.clear();
        tgroups_.clear();
        bool all_ar = true;
        int max_sel = 1;
        for (int i = 0; i < B; ++i) {
            f.attn_kv_unique += hs[i].p + hs[i].nsel;
            f.attn_row_keys += static_cast<double>(hs[i].nsel) * (hs[i].p + 1);
            groups_.push_back(
                {hs[i].vrow_off, hs[i].nsel, hs[i].p, hs[i].p + 1 + std::min(hs[i].l, hs[i].nsel - 1)});
            all_ar = all_ar && hs[i].nsel == 1;
            max_sel = std::max(max_sel, hs[i].nsel);
            // verify rows: committed prefix (p keys; the prompt part from the group leader's
            // copy), paths = the sequence's own verify rows in the scratch region
            const long long cb = static_cast<long long>(hs[i].seq) * tkv_.seq_stride;
            tgroups_.push_back(TreeGroupDev{hs[i].vrow_off, hs[i].nsel, hs[i].p, hs[i].nsel,
                                            tkv_.scratch_base + hs[i].vrow_off, cb, a.g > 1 ? hs[i].pre_base : cb,
                                            a.g > 1 ? std::min(hs[i].pre_len, hs[i].p) : 0, 0});
        }
        f.groups_exact = boundary_tiles();
        // attention_tree.cu for speculative steps, and for AR steps of few rows (one CTA per row
        // and head streams the whole context: no work-list prologue, no partials); wide AR
        // batches keep attention.cu's head-grouped persistent kernel (98 % of HBM at c2)
        static const int tree_ar_max = [] {
            const char* v = getenv("SGB_TREE_AR_MAX");  // A/B switch
            return v ? atoi(v) : 0;
        }();
        // measured (profiles/r02_tree_nst.jsonl, 3-stage ring): attention_tree.cu wins from 3 rows per
        // sequence (48 x 4 rows over 2k keys: 0.274 vs 0.364 ms per layer; 16 x 13: 0.075 vs 0.164;
        // B=1 x 211: 0.057 vs 0.083), attention.cu's shared tiles at 2 (32 x 2 over 4k: 0.372 vs 0.471)
        static const int tree_min_rows = [] {
            const char* v = getenv("SGB_TREE_MIN_ROWS");  // A/B switch
            return v ? atoi(v) : 3;
        }();
        if (((!all_ar && max_sel >= tree_min_rows) || (all_ar && vrows <= tree_ar_max)) && tree_attn_ok(max_sel))
            f.tree = &tgroups_;
        // AR steps of few rows: the cluster decode kernel (attention_tree.cu) spreads each row's
        // key blocks over up to 8 CTAs instead of one warp per row (tree kernel) or attention.cu's
        // global-partials work list
        static const int decode_ar_max = [] {
            // measured crossover vs attention.cu (profiles/r02_decode_attn.jsonl): <= 4 rows
            const char* v = getenv("SGB_DECODE_AR_MAX");  // A/B switch
            return v ? atoi(v) : 4;
        }();
        if (all_ar && vrows <= decode_ar_max) {
            f.tree = &tgroups_;
            f.decode = true;
            f.decode_max_ctx = max_p;
        }
        f.merge_tiles = !all_ar;  // verify tiles of a speculative step (not the AR prompt tiles)
        // measured A/B (SGB_PROMPT_TILES, bench.py vanilla): +5 % at 12 heads (c2), -13 % at
        // 28 heads (c3, where the per-row kernel already hits the prompt pages in L2)
        static const int prompt_tiles = [] {
            const char* v = getenv("SGB_PROMPT_TILES");  // A/B switch
            return v ? atoi(v) : -1;
        }();
        const bool use_prompt_tiles = prompt_tiles < 0 ? dims_.heads <= 16 : prompt_tiles != 0;
        if (all_ar && a.g > 1 && use_prompt_tiles) {
            f.groups_exact = false;  // members share only their prompt
            // AR step: the live members of a query group (consecutive rows) read their prompt's
            // K/V from the leader's copy, so they share the prompt blocks as one tile
            groups_.clear();
            for (int i = 0; i < B;) {
                int j = i + 1, shared = std::min(hs[i].pre_len, hs[i].p), vmax = hs[i].p + 1;
                while (j < B && hs[j].pre_base == hs[i].pre_base) {
                    shared = std::min(shared, std::min(hs[j].pre_len, hs[j].p));
                    vmax = std::max(vmax, hs[j].p + 1);
                    ++j;
                }
                groups_.push_back({hs[i].vrow_off, j - i, shared, vmax});
                i = j;
            }
        }
        f.groups = &groups_;
        forward(f);
        res.target_forwards++;
        // ---- acceptance, walk, commit (scheduler.cpp:219-231)
        nv_phase.reset();
        nv_phase.emplace("sgb accept");
        pe0 = pbeg();
        launch_emit(logits_, V, nullptr, rows_.seed, rows_.key_pos, vrows, a.temperature, emitted_, err_, rsc_, st_);
        count(emit_launches(a.temperature) - 1);
        pend(kClsSample, pe0, 4.0 * vrows * V, 0);
        pe0 = pbeg();
        if (rej && n_spec > 0)
            launch_walk_reject(B, steps_, ss_, tr_, rows_, emitted_, logits_, rsc_.rowmax, qbuf_, qstat_, V,
                               a.temperature, nullptr, acc_rows_, result_, st_);
        else
            launch_walk_commit(B, steps_, ss_, tr_, rows_, emitted_, acc_rows_, result_, st_);
        pend(kClsTree, pe0, 0, 0);
        pe0 = pbeg();
        launch_commit_kv(B, steps_, acc_rows_, result_, tkv_.layers, d, tkv_.K, tkv_.V, tkv_.n_slots * d, tkv_.seq_stride,
                         tkv_.scratch_base, y_, feats_, T, st_);
        pend(kClsCommit, pe0, 0, 0);
        count(3);
        d2h(h_result_, result_, 2 * B, st_);
        d2h(h_result_ + 2 * B, err_, 1, st_);
        SGB_CUDA(cudaEventRecord(evs_b_, st_));
        res.host_enqueue_seconds += std::chrono::duration<double>(std::chrono::steady_clock::now() - t_host0).count();
        SGB_CUDA(cudaStreamSynchronize(st_));
        {
            float ms = 0.f, gap = 0.f;
            SGB_CUDA(cudaEventElapsedTime(&ms, evs_a_, evs_b_));
            SGB_CUDA(cudaEventElapsedTime(&gap, evs_a_, evs_c_));
            res.host_gap_seconds += gap * 1e-3;
            res.step_seconds.push_back(ms * 1e-3);
            std::swap(evs_a_, evs_b_);
        }
        const int err = h_result_[2 * B];
        if (err & 1) throw std::runtime_error("forward_target: non-finite logits");
        if (err & 8) throw std::invalid_argument("build_tree_mask: closure violation");
        pflush();
        for (int i = 0; i < B; ++i) {
            const int s = live[i];
            const int acc = h_result_[2 * i];
            len[s] += acc;
            fin[s] = h_result_[2 * i + 1];
            stat.accepted += acc;
            res.events.push_back(step);
            res.events.push_back(sid_of[s]);
            res.events.push_back(acc);
        }
        res.steps.push_back(stat);
        {
            // SURVEY §8(d) algorithmic work of this step (bf16 weights and K/V): the target
            // forward streams its non-embedding weights once and every sequence's context K/V,
            // writes the verify rows' K/V; each draft pass (catch-up + levels) streams the draft
            // layer + fuse + the shared LM head and the draft context K/V
            const double dd = d, L = mc.layers, Fd = mc.dff, Vv = V;
            const double Pt = L * (4 * dd * dd + 2 * dd * Fd) + dd * Vv;
            const double Pd = dlayers_ * (4 * dd * dd + 2 * dd * Fd) + 2 * dd * dd + dd * Vv;
            const double kvb = 4.0 * L * dd;
            double ctx = 0, rowsN = 0, ctxrows = 0, spec_ctx = 0;
            for (int i = 0; i < B; ++i) {
                ctx += hs[i].p;
                rowsN += hs[i].nsel;
                ctxrows += static_cast<double>(hs[i].nsel) * (hs[i].p + hs[i].nsel);
                if (hs[i].k) spec_ctx += hs[i].p;
            }
            const double passes = n_spec > 0 ? 1.0 + std::max(0, max_l - 1) : 0.0;
            const double bytes = 2 * Pt + ctx * kvb + rowsN * kvb + passes * (2 * Pd + spec_ctx * 4 * dd) +
                                 rowsN * Vv * 4 * (a.temperature > 0 ? 2 : 1);
            const double flops = 2 * Pt * rowsN + 4 * L * dd * ctxrows + 2 * Pd * stat.draft_rows;
            res.step_bytes.push_back(bytes);
            res.step_flops.push_back(flops);
        }
        res.total_accepted += stat.accepted;
        res.total_verify_slots += B;
        if (next_group < P) {  // waves: recycle the regions of finished groups, admit the next groups
            bool freed = false;
            for (int gs = 0; gs < n_gslots; ++gs) {
                if (gslot_group[gs] < 0) continue;
                bool done = true;
                for (int r = 0; r < G && done; ++r) done = fin[gs * G + r] != 0;
                if (!done) continue;
                for (int r = 0; r < G; ++r) retire(gs * G + r);
                gslot_group[gs] = -1;
                freed = true;
            }
            if (freed) {
                SGB_CUDA(cudaStreamSynchronize(st_));
                admit();
                SGB_CUDA(cudaEventRecord(evs_a_, st_));  // the next step is timed after the admission prefill
            }
        }
    }
    SGB_CUDA(cudaEventRecord(ev1_, st_));

    // ---------------- results (scheduler.cpp:343-353) of the sequences still resident
    std::vector<int> h_eos(S);
    d2h(h_eos.data(), ss_.hit_eos, S, st_);
    std::vector<int> resident;
    for (int s2 = 0; s2 < S; ++s2)
        if (sid_of[s2] >= 0) resident.push_back(s2);
    for (int s2 : resident) {
        const int sid = sid_of[s2];
        res.tokens[sid].resize(len[s2]);
        d2h(res.tokens[sid].data(), ss_.tokens + static_cast<size_t>(s2) * T, len[s2], st_);
        sid_len[sid] = len[s2];
    }
    const int slot_hi = resident.empty() ? 0 : resident.back() + 1;
    if (a.want_features && a.features_out && slot_hi > 0) {
        // one DMA of the resident feature store into pinned staging at full link rate ...
        const size_t n = static_cast<size_t>(slot_hi) * T * d;
        if (feats_host_cap_ < n) {
            if (feats_host_) cudaFreeHost(feats_host_);
            feats_host_ = nullptr;
            SGB_CUDA(cudaMallocHost(&feats_host_, n * sizeof(float)));
            feats_host_cap_ = n;
        }
        SGB_CUDA(cudaMemcpyAsync(feats_host_, feats_, n * sizeof(float), cudaMemcpyDeviceToHost, st_));
    } else if (a.want_features) {
        for (int s2 : resident) {
            const int sid = sid_of[s2];
            res.features[sid].resize(static_cast<size_t>(len[s2] - 1) * d);
            d2h(res.features[sid].data(), feats_ + static_cast<size_t>(s2) * T * d, res.features[sid].size(), st_);
        }
    }
    SGB_CUDA(cudaStreamSynchronize(st_));
    if (a.want_features && a.features_out && slot_hi > 0) {
        // ... then the per-sequence scatter into the caller's layout (sid order) on host threads
        const int nth = std::max(1, std::min(16, static_cast<int>(std::thread::hardware_concurrency())));
        std::vector<std::thread> pool;
        const int nres = static_cast<int>(resident.size());
        for (int w = 0; w < nth; ++w)
            pool.emplace_back([&, w] {
                for (int k = w; k < nres; k += nth) {
                    const int s2 = resident[k];
                    std::memcpy(a.features_out + static_cast<size_t>(sid_of[s2]) * (T - 1) * d,
                                feats_host_ + static_cast<size_t>(s2) * T * d,
                                static_cast<size_t>(len[s2] - 1) * d * sizeof(float));
                }
            });
        for (auto& t : pool) t.join();
    }
    for (int s2 : resident) sid_eos[sid_of[s2]] = h_eos[s2];
    res.hit_eos = sid_eos;
    // the draft update / group advantages can consume this rollout straight from HBM when every
    // sequence is still resident at region == sid (no waves)
    last_waves_ = waves;
    if (!waves) {
        last_lens_ = sid_len;
        last_plens_ = res.prompt_len;
    } else {
        last_lens_.clear();
        last_plens_.clear();
    }
    for (int sid = 0; sid < n_seqs; ++sid) {
        res.d2h_bytes += static_cast<long long>(sid_len[sid]) * sizeof(int);
        if (a.want_features) res.d2h_bytes += static_cast<long long>(sid_len[sid] - 1) * d * sizeof(float);
    }
    res.waves = waves;
    float ms = 0.f;
    SGB_CUDA(cudaEventElapsedTime(&ms, ev0_, ev1_));
    res.seconds = ms * 1e-3;
    res.kernel_launches = launches_ - launches0;
    return res;
}

}  // namespace sgb
