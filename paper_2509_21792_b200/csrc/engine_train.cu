// Engine::draft_update -- the online draft-learning step of FastGRPO (grpo.cpp:177-186 /
// grpo.hpp:278-344) on the device. The 1-layer EAGLE-style draft is trained on the
// rollout it just produced, straight from HBM (tokens + target features never leave the
// GPU), with the target LM head frozen:
//
//   forward  (tinylm.hpp:881-921): fuse GEMM -> LN1 -> qkv GEMM -> causal attention ->
//            wo GEMM (+res) -> LN2 -> w1 GEMM -> GELU -> w2 GEMM (+res) -> LNf
//   loss     (grpo.hpp:311-339): SmoothL1(f_hat, f_j)/(rows*d)*w_feat + CE(lm_head f_hat,
//            t_{j+1})/rows*w_tok, the LM head logits computed and consumed in row chunks
//            (never materialised for the whole batch)
//   backward (tinylm.hpp:720-800, 923-953): dgrad GEMMs use the reference-layout bf16
//            weights ([in][out] is the K-major operand for dX = dY.W^T), wgrad GEMMs use
//            transposed activations and accumulate straight into the fp32 gradient in the
//            reference flat layout (epilogue +=)
//   AdamW    (grpo.cpp:142-161) on the fp32 master draft, then bf16 re-conversion.
// All GEMMs are the tcgen05 kernel of gemm.cu; the row kernels live in train.cu.
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <vector>

#include "engine.h"
#include "train.h"
#include "util.h"

namespace sgb {

namespace {
template <class T>
T* talloc(size_t n) {
    T* p = nullptr;
    SGB_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    return p;
}
int pad8(int x) { return (x + 7) & ~7; }
constexpr int kWholeK = 1 << 20;  // one accumulation chunk: training GEMMs have tiles to spare
}  // namespace

void Engine::train_alloc() {
    if (tr2_.ready) return;
    if (dlayers_ != 1) throw std::invalid_argument("draft_update on device supports a 1-layer draft (the reference default)");
    const size_t d = dims_.d, F = dims_.dff, V = dims_.vocab, H = dims_.heads;
    const size_t R = std::max(1024, ((dims_.max_seq + 255) / 256) * 256);  // a whole sequence always fits
    tr2_.rmax = static_cast<int>(R);
    tr2_.lc = static_cast<int>(std::max<size_t>(128, std::min<size_t>(1024, (size_t(1) << 31) / (V * 4))));
    tr2_.smax = dims_.max_seq;
    Train& t = tr2_;
    t.x0 = talloc<float>(R * d);
    t.xmid = talloc<float>(R * d);
    t.xfin = talloc<float>(R * d);
    t.fhat = talloc<float>(R * d);
    t.dlnf = talloc<float>(R * d);
    t.dx = talloc<float>(R * d);
    t.dxmid = talloc<float>(R * d);
    t.dx0 = talloc<float>(R * d);
    t.ctx = talloc<float>(R * d);
    t.dctx = talloc<float>(R * d);
    t.da = talloc<float>(R * d);
    t.qkv = talloc<float>(R * 3 * d);
    t.dqkv = talloc<float>(R * 3 * d);
    t.fch = talloc<float>(R * F);
    t.dhg = talloc<float>(R * F);
    t.dgb = talloc<float>(R * 2 * d);
    t.lse = talloc<float>(R * H);
    t.Drow = talloc<float>(R * H);
    t.mu1 = talloc<float>(R);
    t.rs1 = talloc<float>(R);
    t.mu2 = talloc<float>(R);
    t.rs2 = talloc<float>(R);
    t.muf = talloc<float>(R);
    t.rsf = talloc<float>(R);
    t.logits = talloc<float>(static_cast<size_t>(t.lc) * V);
    t.sc = talloc<float>(R * 2 * static_cast<size_t>(t.smax));
    t.grad = talloc<float>(dlay_.total);
    t.m = talloc<float>(dlay_.total);
    t.v = talloc<float>(dlay_.total);
    SGB_CUDA(cudaMemset(t.m, 0, dlay_.total * 4));
    SGB_CUDA(cudaMemset(t.v, 0, dlay_.total * 4));
    t.fuse = talloc<__nv_bfloat16>(R * 2 * d);
    t.a1 = talloc<__nv_bfloat16>(R * d);
    t.a2 = talloc<__nv_bfloat16>(R * d);
    t.ctx_b = talloc<__nv_bfloat16>(R * d);
    t.fhat_b = talloc<__nv_bfloat16>(R * d);
    t.dx_b = talloc<__nv_bfloat16>(R * d);
    t.dxmid_b = talloc<__nv_bfloat16>(R * d);
    t.hg = talloc<__nv_bfloat16>(R * F);
    t.dfch_b = talloc<__nv_bfloat16>(R * F);
    t.dqkv_b = talloc<__nv_bfloat16>(R * 3 * d);
    t.dlog = talloc<__nv_bfloat16>(static_cast<size_t>(t.lc) * V);
    const size_t tmax = std::max({2 * d, 3 * d, F});
    t.tA = talloc<__nv_bfloat16>(tmax * R);
    t.tB = talloc<__nv_bfloat16>(tmax * R);
    t.dflat_b = talloc<__nv_bfloat16>(dlay_.total);
    t.wqkv_ref = talloc<__nv_bfloat16>(3 * d * d);
    t.lm_ref = talloc<__nv_bfloat16>(d * V);
    t.tok = talloc<int>(R);
    t.pos = talloc<int>(R);
    t.next = talloc<int>(R);
    t.seq_first = talloc<int>(R);
    t.seq_last = talloc<int>(R);
    t.tiles = talloc<int>(R);
    t.prev_off = talloc<long long>(R);
    t.tgt_off = talloc<long long>(R);
    t.loss_row = talloc<double>(2 * R);
    t.feat_in = nullptr;
    const int Ri = static_cast<int>(R);
    t.act_fuse.init(t.fuse, Ri, 2 * d);
    t.act_a1.init(t.a1, Ri, d);
    t.act_a2.init(t.a2, Ri, d);
    t.act_ctx.init(t.ctx_b, Ri, d);
    t.act_hg.init(t.hg, Ri, F);
    t.act_dx.init(t.dx_b, Ri, d);
    t.act_dxmid.init(t.dxmid_b, Ri, d);
    t.act_dfch.init(t.dfch_b, Ri, F);
    t.act_dqkv.init(t.dqkv_b, Ri, 3 * d);
    t.act_dlog.init(t.dlog, t.lc, V);
    // frozen target LM head in the reference layout [d][V] (K-major operand of its dgrad)
    launch_transpose_bf16(lm_head_.ptr, static_cast<int>(V), static_cast<int>(d), static_cast<int>(d), t.lm_ref,
                          static_cast<int>(V), st_);
    t.lm_ref_w.init(t.lm_ref, d, V, kWholeK);
    t.ready = true;
    train_refresh_ref_weights();
}

void Engine::adamw_reset() {
    if (!tr2_.ready) return;
    SGB_CUDA(cudaMemsetAsync(tr2_.m, 0, dlay_.total * 4, st_));
    SGB_CUDA(cudaMemsetAsync(tr2_.v, 0, dlay_.total * 4, st_));
    tr2_.adam_t = 0;
}

// AdamW moments + step count (grpo.hpp:97-103) between the device and a caller's AdamW object:
// upload (m, v nullptr = a fresh optimizer's zeros) or download.
void Engine::adamw_state(float* m, float* v, long long* t, bool upload) {
    if (!target_ready_ || !draft_ready_) throw std::runtime_error("weights not uploaded");
    train_alloc();
    const size_t n = dlay_.total;
    if (upload) {
        if (m) SGB_CUDA(cudaMemcpyAsync(tr2_.m, m, n * 4, cudaMemcpyHostToDevice, st_));
        else SGB_CUDA(cudaMemsetAsync(tr2_.m, 0, n * 4, st_));
        if (v) SGB_CUDA(cudaMemcpyAsync(tr2_.v, v, n * 4, cudaMemcpyHostToDevice, st_));
        else SGB_CUDA(cudaMemsetAsync(tr2_.v, 0, n * 4, st_));
        tr2_.adam_t = t ? *t : 0;
    } else {
        if (m) SGB_CUDA(cudaMemcpyAsync(m, tr2_.m, n * 4, cudaMemcpyDeviceToHost, st_));
        if (v) SGB_CUDA(cudaMemcpyAsync(v, tr2_.v, n * 4, cudaMemcpyDeviceToHost, st_));
        if (t) *t = tr2_.adam_t;
    }
    SGB_CUDA(cudaStreamSynchronize(st_));
}

// bf16 copies of the draft master in the reference [in][out] layout: the K-major operands
// of the dgrad GEMMs (dX = dY . W^T).
void Engine::train_refresh_ref_weights() {
    Train& t = tr2_;
    const size_t d = dims_.d, F = dims_.dff;
    launch_f32_to_bf16(dmaster_, dlay_.total, t.dflat_b, st_);
    const auto& o = dlay_.layers[0];
    for (int k = 0; k < 3; ++k) {
        const size_t off = k == 0 ? o.wq : (k == 1 ? o.wk : o.wv);
        SGB_CUDA(cudaMemcpy2DAsync(t.wqkv_ref + k * d, 3 * d * 2, t.dflat_b + off, d * 2, d * 2, d,
                                   cudaMemcpyDeviceToDevice, st_));
    }
    t.wqkv_ref_w.init(t.wqkv_ref, d, 3 * d, kWholeK);
    t.wo_ref.init(t.dflat_b + o.wo, d, d, kWholeK);
    t.w1_ref.init(t.dflat_b + o.w1, d, F, kWholeK);
    t.w2_ref.init(t.dflat_b + o.w2, F, d, kWholeK);
}

// grad[k][n] (+)= sum_r X[r][k] dY[r][n], from transposed operands dyT [N][Rp], xT [Kfeat][Rp].
void Engine::wgrad(const __nv_bfloat16* dyT, int N, const __nv_bfloat16* xT, int Kfeat, int Rp, float* grad_dst,
                   int ld) {
    GemmWeight w;
    w.init(dyT, N, Rp, kWholeK);
    GemmAct a;
    a.init(xT, Kfeat, Rp);
    GemmEpi e;
    e.kind = kEpiResid;
    e.f32 = grad_dst;
    e.ld = ld;
    gemm(w, a, Kfeat, e, kClsGemm, 4.0);
}

Engine::DraftLossTerms Engine::draft_update(const DraftUpdateArgs& A) {
    NvtxRange nv("sgb draft_update");
    if (!target_ready_ || !draft_ready_) throw std::runtime_error("weights not uploaded");
    train_alloc();
    Train& t = tr2_;
    if (draft_lm_stale_) {  // the target's LM head changed (policy update / re-upload)
        launch_transpose_bf16(lm_head_.ptr, dims_.vocab, dims_.d, dims_.d, t.lm_ref, dims_.vocab, st_);
        draft_lm_stale_ = false;
    }
    const int d = dims_.d, F = dims_.dff, V = dims_.vocab, H = dims_.heads;
    const auto& lo = dlay_.layers[0];
    const LayerDev& W = dL_[0];
    DraftLossTerms terms;
    struct Ev {  // RAII: no leaked events on early return / exception
        cudaEvent_t e = nullptr;
        Ev() { SGB_CUDA(cudaEventCreate(&e)); }
        ~Ev() { cudaEventDestroy(e); }
    } ev0, ev1;
    cudaEvent_t e0 = ev0.e, e1 = ev1.e;
    SGB_CUDA(cudaEventRecord(e0, st_));

    // ---- sequence table + feature source
    std::vector<int> lens;
    std::vector<long long> tok_off, feat_off;  // per sequence
    const float* feat_base = nullptr;
    const int* tok_base_dev = nullptr;
    std::vector<int> host_tokens;
    if (A.use_last_rollout) {
        if (last_waves_) throw std::invalid_argument("draft_update: the last rollout ran in waves (not resident in HBM)");
        lens = last_lens_;
        for (size_t s = 0; s < lens.size(); ++s) {
            tok_off.push_back(static_cast<long long>(s) * dims_.max_seq);
            feat_off.push_back(static_cast<long long>(s) * dims_.max_seq * d);
        }
        feat_base = feats_;
        tok_base_dev = ss_.tokens;
    } else {
        lens.assign(A.lens, A.lens + A.n_seqs);
        long long to = 0, fo = 0;
        for (int L : lens) {
            if (L < 0 || L > dims_.max_seq) throw std::invalid_argument("draft_update: bad sequence length");
            tok_off.push_back(to);
            feat_off.push_back(fo);
            to += L;
            fo += static_cast<long long>(std::max(0, L - 1)) * d;
        }
        if (static_cast<size_t>(fo) > t.feat_cap) {
            if (t.feat_in) cudaFree(t.feat_in);
            t.feat_in = talloc<float>(fo);
            t.feat_cap = fo;
        }
        SGB_CUDA(cudaMemcpyAsync(t.feat_in, A.features, fo * 4, cudaMemcpyHostToDevice, st_));
        feat_base = t.feat_in;
        host_tokens.assign(A.tokens, A.tokens + to);
    }
    long long rows_local = 0;
    for (int L : lens) rows_local += std::max(0, L - 2);
    terms.rows = rows_local;
    const long long rows_norm = A.rows_total > 0 ? A.rows_total : rows_local;
    SGB_CUDA(cudaMemsetAsync(t.grad, 0, dlay_.total * 4, st_));
    if (lens.empty() || rows_norm == 0) {
        // a data-parallel rank with no rows still joins the gradient all-reduce (zero
        // contribution), or the other ranks would wait in ncclAllReduce forever
        if (A.grad_hook) A.grad_hook(t.grad, dlay_.total, st_, A.hook_ctx);
        SGB_CUDA(cudaStreamSynchronize(st_));
        return terms;
    }
    const double inv_r = 1.0 / static_cast<double>(rows_norm);
    const double scale_feat = A.w_feat * inv_r / d, scale_tok = A.w_tok * inv_r;

    // host tokens of the last rollout are needed to build the row tables
    std::vector<int> dev_tok_copy;
    if (A.use_last_rollout) {
        dev_tok_copy.resize(lens.size() * static_cast<size_t>(dims_.max_seq));
        SGB_CUDA(cudaMemcpyAsync(dev_tok_copy.data(), tok_base_dev, dev_tok_copy.size() * 4, cudaMemcpyDeviceToHost, st_));
        SGB_CUDA(cudaStreamSynchronize(st_));
    }
    const int* htok = A.use_last_rollout ? dev_tok_copy.data() : host_tokens.data();

    // ---- chunks of whole sequences
    size_t s_begin = 0;
    std::vector<double> hloss;
    while (s_begin < lens.size()) {
        std::vector<int> tok, pos, next, sfirst, slast, tiles;
        std::vector<long long> poff, toff;
        size_t s = s_begin;
        for (; s < lens.size(); ++s) {
            const int rows = std::max(0, lens[s] - 2);
            if (!tok.empty() && static_cast<int>(tok.size()) + rows > t.rmax) break;
            if (rows > t.rmax) throw std::invalid_argument("draft_update: sequence longer than the training chunk");
            const int first = static_cast<int>(tok.size());
            for (int m = 0; m < rows; m += 64) tiles.push_back(first + m);  // attention tiles per sequence
            for (int j = 1; j <= rows; ++j) {  // pair (t_j, f_{j-1}) -> targets (f_j, t_{j+1})
                tok.push_back(htok[tok_off[s] + j]);
                pos.push_back(j);
                next.push_back(htok[tok_off[s] + j + 1]);
                poff.push_back(feat_off[s] + static_cast<long long>(j - 1) * d);
                toff.push_back(feat_off[s] + static_cast<long long>(j) * d);
                sfirst.push_back(first);
                slast.push_back(first + rows - 1);
            }
        }
        s_begin = s;
        const int R = static_cast<int>(tok.size());
        if (R == 0) continue;
        const int Rp = pad8(R);
        SGB_CUDA(cudaMemcpyAsync(t.tok, tok.data(), R * 4, cudaMemcpyHostToDevice, st_));
        SGB_CUDA(cudaMemcpyAsync(t.pos, pos.data(), R * 4, cudaMemcpyHostToDevice, st_));
        SGB_CUDA(cudaMemcpyAsync(t.next, next.data(), R * 4, cudaMemcpyHostToDevice, st_));
        SGB_CUDA(cudaMemcpyAsync(t.seq_first, sfirst.data(), R * 4, cudaMemcpyHostToDevice, st_));
        SGB_CUDA(cudaMemcpyAsync(t.seq_last, slast.data(), R * 4, cudaMemcpyHostToDevice, st_));
        const int n_tiles = static_cast<int>(tiles.size());
        SGB_CUDA(cudaMemcpyAsync(t.tiles, tiles.data(), n_tiles * 4, cudaMemcpyHostToDevice, st_));
        SGB_CUDA(cudaMemcpyAsync(t.prev_off, poff.data(), R * 8, cudaMemcpyHostToDevice, st_));
        SGB_CUDA(cudaMemcpyAsync(t.tgt_off, toff.data(), R * 8, cudaMemcpyHostToDevice, st_));

        // ---------------- forward with saved activations (tinylm.hpp:881-921, 653-718)
        launch_gather_fuse(t.tok, t.prev_off, feat_base, tok_emb_, R, d, t.fuse, st_);
        GemmEpi e;
        e.kind = kEpiFusePos;
        e.f32 = t.x0;
        e.pos_emb = pos_emb_;
        e.pos = t.pos;
        e.ld = d;
        gemm(w_fuse_, t.act_fuse, R, e, kClsGemm, 8.0);
        launch_ln_fwd_stats(t.x0, R, d, W.ln1_g, W.ln1_b, t.a1, nullptr, t.mu1, t.rs1, st_);
        e = GemmEpi{};
        e.kind = kEpiF32;
        e.f32 = t.qkv;
        e.ld = 3 * d;
        gemm(W.qkv, t.act_a1, R, e, kClsGemm, 4.0);
        launch_train_attn_fwd(t.qkv, t.seq_first, t.seq_last, t.tiles, n_tiles, d, H, t.ctx, t.ctx_b, t.lse, st_);
        SGB_CUDA(cudaMemcpyAsync(t.xmid, t.x0, static_cast<size_t>(R) * d * 4, cudaMemcpyDeviceToDevice, st_));
        e = GemmEpi{};
        e.kind = kEpiResid;
        e.f32 = t.xmid;
        e.ld = d;
        gemm(W.wo, t.act_ctx, R, e, kClsGemm, 8.0);
        launch_ln_fwd_stats(t.xmid, R, d, W.ln2_g, W.ln2_b, t.a2, nullptr, t.mu2, t.rs2, st_);
        e = GemmEpi{};
        e.kind = kEpiF32;
        e.f32 = t.fch;
        e.ld = F;
        gemm(W.w1, t.act_a2, R, e, kClsGemm, 4.0);
        launch_gelu_fwd(t.fch, static_cast<size_t>(R) * F, t.hg, st_);
        SGB_CUDA(cudaMemcpyAsync(t.xfin, t.xmid, static_cast<size_t>(R) * d * 4, cudaMemcpyDeviceToDevice, st_));
        e = GemmEpi{};
        e.kind = kEpiResid;
        e.f32 = t.xfin;
        e.ld = d;
        gemm(W.w2, t.act_hg, R, e, kClsGemm, 8.0);
        launch_ln_fwd_stats(t.xfin, R, d, dlnf_g_, dlnf_b_, t.fhat_b, t.fhat, t.muf, t.rsf, st_);

        // ---------------- losses (grpo.hpp:311-339)
        launch_smoothl1(t.fhat, feat_base, t.tgt_off, R, d, scale_feat, t.dlnf, t.loss_row, st_);
        for (int r0 = 0; r0 < R; r0 += t.lc) {
            const int rc = std::min(t.lc, R - r0);
            GemmAct af;
            af.init(t.fhat_b + static_cast<size_t>(r0) * d, rc, d);
            e = GemmEpi{};
            e.kind = kEpiF32;
            e.f32 = t.logits;
            e.ld = V;
            gemm(lm_head_, af, rc, e, kClsLmHead, 4.0);
            launch_ce(t.logits, rc, V, t.next + r0, scale_tok, t.dlog, t.loss_row + R + r0, st_);
            // d_lnf += dlogits . lm_head^T   (tinylm.hpp:940-943)
            e = GemmEpi{};
            e.kind = kEpiResid;
            e.f32 = t.dlnf + static_cast<size_t>(r0) * d;
            e.ld = d;
            gemm(t.lm_ref_w, t.act_dlog, rc, e, kClsLmHead, 8.0);
        }
        {
            std::vector<double> lr(2 * R);
            SGB_CUDA(cudaMemcpyAsync(lr.data(), t.loss_row, 2 * R * 8, cudaMemcpyDeviceToHost, st_));
            SGB_CUDA(cudaStreamSynchronize(st_));
            for (int r = 0; r < R; ++r) terms.feature_loss += lr[r];
            for (int r = 0; r < R; ++r) terms.token_loss += lr[R + r];
        }

        // ---------------- backward (tinylm.hpp:923-953, 720-800)
        launch_ln_bwd(t.xfin, dlnf_g_, t.muf, t.rsf, t.dlnf, nullptr, R, d, t.dx, t.dgb, st_);
        launch_colsum_add(t.dgb, R, 2 * d, t.grad + dlay_.lnf_g, st_);
        // MLP: dW2 += hg^T dx ; d_hg = dx W2^T ; gelu' ; dW1 += a2^T dfch ; d_a2 = dfch W1^T
        launch_transpose_bf16(t.dx, R, d, d, t.tA, Rp, st_);
        launch_transpose_bf16(t.hg, R, F, F, t.tB, Rp, st_);
        wgrad(t.tA, d, t.tB, F, Rp, t.grad + lo.w2, d);
        launch_f32_to_bf16(t.dx, static_cast<size_t>(R) * d, t.dx_b, st_);
        e = GemmEpi{};
        e.kind = kEpiF32;
        e.f32 = t.dhg;
        e.ld = F;
        gemm(t.w2_ref, t.act_dx, R, e, kClsGemm, 4.0);
        launch_gelu_bwd(t.fch, t.dhg, static_cast<size_t>(R) * F, t.dfch_b, st_);
        launch_transpose_bf16(t.dfch_b, R, F, F, t.tA, Rp, st_);
        launch_transpose_bf16(t.a2, R, d, d, t.tB, Rp, st_);
        wgrad(t.tA, F, t.tB, d, Rp, t.grad + lo.w1, F);
        e = GemmEpi{};
        e.kind = kEpiF32;
        e.f32 = t.da;
        e.ld = d;
        gemm(t.w1_ref, t.act_dfch, R, e, kClsGemm, 4.0);
        launch_ln_bwd(t.xmid, W.ln2_g, t.mu2, t.rs2, t.da, t.dx, R, d, t.dxmid, t.dgb, st_);
        launch_colsum_add(t.dgb, R, 2 * d, t.grad + lo.ln2_g, st_);
        // attention: dWo += ctx^T dxmid ; dctx = dxmid Wo^T ; attention bwd ; dWq/k/v ; d_a1
        launch_transpose_bf16(t.dxmid, R, d, d, t.tA, Rp, st_);
        launch_transpose_bf16(t.ctx_b, R, d, d, t.tB, Rp, st_);
        wgrad(t.tA, d, t.tB, d, Rp, t.grad + lo.wo, d);
        launch_f32_to_bf16(t.dxmid, static_cast<size_t>(R) * d, t.dxmid_b, st_);
        e = GemmEpi{};
        e.kind = kEpiF32;
        e.f32 = t.dctx;
        e.ld = d;
        gemm(t.wo_ref, t.act_dxmid, R, e, kClsGemm, 4.0);
        launch_train_attn_bwd(t.qkv, t.ctx, t.dctx, t.lse, t.seq_first, t.seq_last, t.tiles, n_tiles, R, d, H, t.Drow,
                              t.dqkv, st_);
        launch_transpose_bf16(t.a1, R, d, d, t.tB, Rp, st_);
        const size_t qkv_off[3] = {lo.wq, lo.wk, lo.wv};
        for (int k = 0; k < 3; ++k) {
            launch_transpose_bf16(t.dqkv + static_cast<size_t>(k) * d, R, d, 3 * d, t.tA, Rp, st_);
            wgrad(t.tA, d, t.tB, d, Rp, t.grad + qkv_off[k], d);
        }
        launch_f32_to_bf16(t.dqkv, static_cast<size_t>(R) * 3 * d, t.dqkv_b, st_);
        e = GemmEpi{};
        e.kind = kEpiF32;
        e.f32 = t.da;
        e.ld = d;
        gemm(t.wqkv_ref_w, t.act_dqkv, R, e, kClsGemm, 4.0);
        launch_ln_bwd(t.x0, W.ln1_g, t.mu1, t.rs1, t.da, t.dxmid, R, d, t.dx0, t.dgb, st_);
        launch_colsum_add(t.dgb, R, 2 * d, t.grad + lo.ln1_g, st_);
        // fuse projection (tinylm.hpp:951-952): dW_fuse += fused^T dx0
        launch_transpose_bf16(t.dx0, R, d, d, t.tA, Rp, st_);
        launch_transpose_bf16(t.fuse, R, 2 * d, 2 * d, t.tB, Rp, st_);
        wgrad(t.tA, d, t.tB, 2 * d, Rp, t.grad + dlay_.w_fuse, d);
        count(40);
    }
    terms.total = terms.feature_loss + terms.token_loss;
    if (A.grad_hook) A.grad_hook(t.grad, dlay_.total, st_, A.hook_ctx);
    if (A.grad_out) {
        SGB_CUDA(cudaMemcpyAsync(A.grad_out, t.grad, dlay_.total * 4, cudaMemcpyDeviceToHost, st_));
    }
    if (A.apply_step) {
        ++t.adam_t;
        launch_adamw(dmaster_, t.grad, t.m, t.v, dlay_.total, A.lr, A.beta1, A.beta2, A.eps, A.weight_decay, t.adam_t,
                     st_);
        convert_draft();
        train_refresh_ref_weights();
    }
    SGB_CUDA(cudaEventRecord(e1, st_));
    SGB_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    SGB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    terms.seconds = ms * 1e-3;
    return terms;
}

}  // namespace sgb
