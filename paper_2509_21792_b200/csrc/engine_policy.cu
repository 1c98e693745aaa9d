// Engine::policy_update -- the GRPO policy step (policy_update, grpo.cpp:163-175 ->
// policy_loss_grad, grpo.hpp:235-276 -> target_train_forward / target_train_backward,
// tinylm.hpp:804-866 -> AdamW::step, grpo.cpp:142-161) on the device, so a training loop never
// moves the target between host and GPU: the fp32 master copy, its gradient and the AdamW
// moments live in HBM next to the bf16 inference weights, which are re-derived after the step.
//
//   forward  x0 = tok_emb[t] + pos_emb[i]; L pre-LN blocks with saved activations (the
//            draft-update kernels of train.cu / train_attn.cu, per layer); final LN; logits in
//            row chunks through the LM head (never materialised for the whole batch)
//   loss     -(1/N) sum_seq sum_{i >= prompt_len} A_seq * log p(t_i | t_<i): the CE kernel with a
//            per-row scale A_seq / N on response rows and 0 on prompt rows
//   backward LM head (trainable here: its wgrad is a V-wide GEMM per chunk), final LN, the
//            blocks in reverse, embeddings (scatter-add into tok_emb / pos_emb rows)
//   AdamW    on the fp32 master, then bf16 re-conversion (convert_target)
// All GEMMs are the tcgen05 kernel of gemm.cu; the dgrad operands are bf16 copies of the master
// in the reference [in][out] layout (K-major for dX = dY . W^T).
#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <vector>

#include "engine.h"
#include "train.h"
#include "util.h"

namespace sgb {

namespace {
std::vector<void*>* g_pol_ptrs = nullptr;  // the allocating engine's list (freed in ~Engine)
template <class T>
T* palloc(size_t n) {
    T* p = nullptr;
    SGB_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    if (g_pol_ptrs) g_pol_ptrs->push_back(p);
    return p;
}
int pad8(int x) { return (x + 7) & ~7; }
constexpr int kWholeK = 1 << 20;
}  // namespace

void Engine::policy_enable() { keep_master_ = true; }

void Engine::download_target(float* flat, size_t n) {
    if (n != tlay_.total) throw std::invalid_argument("download_target: param count mismatch");
    if (!tmaster_) throw std::runtime_error("download_target: no fp32 target master (policy updates not enabled)");
    SGB_CUDA(cudaStreamSynchronize(st_));
    SGB_CUDA(cudaMemcpy(flat, tmaster_, n * sizeof(float), cudaMemcpyDeviceToHost));
}

void Engine::policy_alloc() {
    Pol& p = pol_;
    if (p.ready) return;
    if (!tmaster_) throw std::runtime_error("policy_update: call policy_enable before uploading the target");
    g_pol_ptrs = &pol_ptrs_;
    const size_t d = dims_.d, F = dims_.dff, V = dims_.vocab, H = dims_.heads, Ln = dims_.layers;
    const size_t R = std::max(1024, ((dims_.max_seq + 255) / 256) * 256);
    p.rmax = static_cast<int>(R);
    p.lc = static_cast<int>(std::max<size_t>(128, std::min<size_t>(1024, (size_t(1) << 31) / (V * 4))));
    const size_t P = tlay_.total;
    p.grad = palloc<float>(P);
    p.m = palloc<float>(P);
    p.v = palloc<float>(P);
    SGB_CUDA(cudaMemset(p.m, 0, P * 4));
    SGB_CUDA(cudaMemset(p.v, 0, P * 4));
    p.flat_b = palloc<__nv_bfloat16>(P);
    p.wqkv_ref = palloc<__nv_bfloat16>(Ln * 3 * d * d);
    p.L.resize(Ln);
    const int Ri = static_cast<int>(R);
    for (size_t l = 0; l < Ln; ++l) {
        Pol::Layer& a = p.L[l];
        a.x_in = palloc<float>(R * d);
        a.a1 = palloc<__nv_bfloat16>(R * d);
        a.mu1 = palloc<float>(R);
        a.rs1 = palloc<float>(R);
        a.qkv = palloc<float>(R * 3 * d);
        a.ctx = palloc<float>(R * d);
        a.ctxb = palloc<__nv_bfloat16>(R * d);
        a.lse = palloc<float>(R * H);
        a.xmid = palloc<float>(R * d);
        a.a2 = palloc<__nv_bfloat16>(R * d);
        a.mu2 = palloc<float>(R);
        a.rs2 = palloc<float>(R);
        a.fch = palloc<float>(R * F);
        a.hg = palloc<__nv_bfloat16>(R * F);
        a.act_a1.init(a.a1, Ri, d);
        a.act_ctx.init(a.ctxb, Ri, d);
        a.act_a2.init(a.a2, Ri, d);
        a.act_hg.init(a.hg, Ri, F);
    }
    p.xfin = palloc<float>(R * d);
    p.fhat = palloc<float>(R * d);
    p.fhat_b = palloc<__nv_bfloat16>(R * d);
    p.muf = palloc<float>(R);
    p.rsf = palloc<float>(R);
    p.dlnf = palloc<float>(R * d);
    p.dx = palloc<float>(R * d);
    p.dxmid = palloc<float>(R * d);
    p.da = palloc<float>(R * d);
    p.dctx = palloc<float>(R * d);
    p.dqkv = palloc<float>(R * 3 * d);
    p.dhg = palloc<float>(R * F);
    p.dgb = palloc<float>(R * 2 * d);
    p.Drow = palloc<float>(R * H);
    p.dfch_b = palloc<__nv_bfloat16>(R * F);
    p.dx_b = palloc<__nv_bfloat16>(R * d);
    p.dxmid_b = palloc<__nv_bfloat16>(R * d);
    p.dqkv_b = palloc<__nv_bfloat16>(R * 3 * d);
    p.logits = palloc<float>(static_cast<size_t>(p.lc) * V);
    p.dlog = palloc<__nv_bfloat16>(static_cast<size_t>(p.lc) * V);
    const size_t tmax = std::max({3 * d * R, F * R, V * static_cast<size_t>(pad8(p.lc))});
    p.tA = palloc<__nv_bfloat16>(tmax);
    p.tB = palloc<__nv_bfloat16>(std::max(F, 3 * d) * R);
    p.tok = palloc<int>(R);
    p.pos = palloc<int>(R);
    p.next = palloc<int>(R);
    p.seq_first = palloc<int>(R);
    p.seq_last = palloc<int>(R);
    p.tiles = palloc<int>(R);
    p.rscale = palloc<double>(R);
    p.csr = palloc<int>(3 * R + 2);
    p.loss_row = palloc<double>(R);
    p.act_fhat.init(p.fhat_b, Ri, d);
    p.act_dx.init(p.dx_b, Ri, d);
    p.act_dxmid.init(p.dxmid_b, Ri, d);
    p.act_dfch.init(p.dfch_b, Ri, F);
    p.act_dqkv.init(p.dqkv_b, Ri, 3 * d);
    p.act_dlog.init(p.dlog, p.lc, V);
    p.ready = true;
    g_pol_ptrs = nullptr;
    policy_refresh_ref_weights();
}

// bf16 copies of the master in the reference [in][out] layout (dgrad operands), wq|wk|wv
// interleaved per input row for the fused dX = dQKV . Wqkv^T
void Engine::policy_refresh_ref_weights() {
    Pol& p = pol_;
    const size_t d = dims_.d, F = dims_.dff, V = dims_.vocab;
    launch_f32_to_bf16(tmaster_, tlay_.total, p.flat_b, st_);
    p.refs.resize(dims_.layers);
    for (int l = 0; l < dims_.layers; ++l) {
        const auto& o = tlay_.layers[l];
        __nv_bfloat16* q = p.wqkv_ref + static_cast<size_t>(l) * 3 * d * d;
        for (int k = 0; k < 3; ++k) {
            const size_t off = k == 0 ? o.wq : (k == 1 ? o.wk : o.wv);
            SGB_CUDA(cudaMemcpy2DAsync(q + k * d, 3 * d * 2, p.flat_b + off, d * 2, d * 2, d, cudaMemcpyDeviceToDevice, st_));
        }
        Pol::Refs& r = p.refs[l];
        r.wqkv.init(q, d, 3 * d, kWholeK);
        r.wo.init(p.flat_b + o.wo, d, d, kWholeK);
        r.w1.init(p.flat_b + o.w1, d, F, kWholeK);
        r.w2.init(p.flat_b + o.w2, F, d, kWholeK);
    }
    p.lm_ref.init(p.flat_b + tlay_.lm_head, d, V, kWholeK);
}

Engine::PolicyTerms Engine::policy_update(const PolicyArgs& A) {
    NvtxRange nv("sgb policy_update");
    if (!target_ready_) throw std::runtime_error("weights not uploaded");
    policy_alloc();
    Pol& p = pol_;
    const int d = dims_.d, F = dims_.dff, V = dims_.vocab, H = dims_.heads, Ln = dims_.layers;
    PolicyTerms terms;
    struct Ev {
        cudaEvent_t e = nullptr;
        Ev() { SGB_CUDA(cudaEventCreate(&e)); }
        ~Ev() { cudaEventDestroy(e); }
    } ev0, ev1;
    SGB_CUDA(cudaEventRecord(ev0.e, st_));

    // ---- sequences (TrainSeq: tokens, prompt_len, weight = advantage; grpo.hpp:66-77)
    std::vector<long long> tok_off(A.n_seqs);
    long long to = 0, n_tokens = 0;
    for (int s = 0; s < A.n_seqs; ++s) {
        const int n = A.lens[s];
        if (n < 0 || n > dims_.max_seq) throw std::invalid_argument("target_train_forward: bad sequence length");
        if (A.prompt_lens[s] < 0 || A.prompt_lens[s] > n) throw std::invalid_argument("policy_update: bad prompt length");
        tok_off[s] = to;
        to += n;
        n_tokens += std::max(0, n - A.prompt_lens[s]);
        for (int i = 0; i < n; ++i)
            if (A.tokens[tok_off[s] + i] < 0 || A.tokens[tok_off[s] + i] >= V)
                throw std::invalid_argument("target_train_forward: token id out of range");
    }
    terms.tokens = n_tokens;
    const long long n_norm = A.tokens_total > 0 ? A.tokens_total : n_tokens;
    SGB_CUDA(cudaMemsetAsync(p.grad, 0, tlay_.total * 4, st_));
    if (n_norm == 0) {  // policy_loss_grad returns 0 with a zero gradient (grpo.hpp:243)
        if (A.grad_hook) A.grad_hook(p.grad, tlay_.total, st_, A.hook_ctx);
        SGB_CUDA(cudaStreamSynchronize(st_));
        terms.skipped = true;
        return terms;
    }
    const double inv_n = 1.0 / static_cast<double>(n_norm);

    size_t s_begin = 0;
    const size_t ns = static_cast<size_t>(A.n_seqs);
    while (s_begin < ns) {
        // ---- a chunk of whole sequences: rows = n - 1 per sequence with a response
        std::vector<int> tok, pos, next, sfirst, slast, tiles;
        std::vector<double> rsc;
        size_t s = s_begin;
        for (; s < ns; ++s) {
            const int n = A.lens[s], q = A.prompt_lens[s];
            if (n - q <= 0) continue;  // grpo.hpp:249
            const int rows = n - 1;
            if (!tok.empty() && static_cast<int>(tok.size()) + rows > p.rmax) break;
            if (rows > p.rmax) throw std::invalid_argument("policy_update: sequence longer than the training chunk");
            const int first = static_cast<int>(tok.size());
            for (int m = 0; m < rows; m += 64) tiles.push_back(first + m);
            const int* t = A.tokens + tok_off[s];
            for (int i = 0; i < rows; ++i) {  // row i scores token i + 1 (grpo.hpp:252-253)
                tok.push_back(t[i]);
                pos.push_back(i);
                next.push_back(t[i + 1]);
                sfirst.push_back(first);
                slast.push_back(first + rows - 1);
                rsc.push_back(i + 1 >= q ? A.weights[s] * inv_n : 0.0);
            }
        }
        s_begin = s;
        const int R = static_cast<int>(tok.size());
        if (R == 0) continue;
        terms.rows += R;
        const int Rp = pad8(R);
        SGB_CUDA(cudaMemcpyAsync(p.tok, tok.data(), R * 4, cudaMemcpyHostToDevice, st_));
        SGB_CUDA(cudaMemcpyAsync(p.pos, pos.data(), R * 4, cudaMemcpyHostToDevice, st_));
        SGB_CUDA(cudaMemcpyAsync(p.next, next.data(), R * 4, cudaMemcpyHostToDevice, st_));
        SGB_CUDA(cudaMemcpyAsync(p.seq_first, sfirst.data(), R * 4, cudaMemcpyHostToDevice, st_));
        SGB_CUDA(cudaMemcpyAsync(p.seq_last, slast.data(), R * 4, cudaMemcpyHostToDevice, st_));
        const int n_tiles = static_cast<int>(tiles.size());
        SGB_CUDA(cudaMemcpyAsync(p.tiles, tiles.data(), n_tiles * 4, cudaMemcpyHostToDevice, st_));
        SGB_CUDA(cudaMemcpyAsync(p.rscale, rsc.data(), R * 8, cudaMemcpyHostToDevice, st_));

        // ---------------- forward with saved activations (tinylm.hpp:804-827, 653-718)
        launch_embed_sum(p.tok, p.pos, R, d, tok_emb_, pos_emb_, p.L[0].x_in, st_);
        for (int l = 0; l < Ln; ++l) {
            Pol::Layer& a = p.L[l];
            const LayerDev& W = tL_[l];
            launch_ln_fwd_stats(a.x_in, R, d, W.ln1_g, W.ln1_b, a.a1, nullptr, a.mu1, a.rs1, st_);
            GemmEpi e;
            e.kind = kEpiF32;
            e.f32 = a.qkv;
            e.ld = 3 * d;
            gemm(W.qkv, a.act_a1, R, e, kClsGemm, 4.0);
            launch_train_attn_fwd(a.qkv, p.seq_first, p.seq_last, p.tiles, n_tiles, d, H, a.ctx, a.ctxb, a.lse, st_);
            SGB_CUDA(cudaMemcpyAsync(a.xmid, a.x_in, static_cast<size_t>(R) * d * 4, cudaMemcpyDeviceToDevice, st_));
            e = GemmEpi{};
            e.kind = kEpiResid;
            e.f32 = a.xmid;
            e.ld = d;
            gemm(W.wo, a.act_ctx, R, e, kClsGemm, 8.0);
            launch_ln_fwd_stats(a.xmid, R, d, W.ln2_g, W.ln2_b, a.a2, nullptr, a.mu2, a.rs2, st_);
            e = GemmEpi{};
            e.kind = kEpiF32;
            e.f32 = a.fch;
            e.ld = F;
            gemm(W.w1, a.act_a2, R, e, kClsGemm, 4.0);
            launch_gelu_fwd(a.fch, static_cast<size_t>(R) * F, a.hg, st_);
            float* xo = l + 1 < Ln ? p.L[l + 1].x_in : p.xfin;
            SGB_CUDA(cudaMemcpyAsync(xo, a.xmid, static_cast<size_t>(R) * d * 4, cudaMemcpyDeviceToDevice, st_));
            e = GemmEpi{};
            e.kind = kEpiResid;
            e.f32 = xo;
            e.ld = d;
            gemm(W.w2, a.act_hg, R, e, kClsGemm, 8.0);
        }
        launch_ln_fwd_stats(p.xfin, R, d, lnf_g_, lnf_b_, p.fhat_b, p.fhat, p.muf, p.rsf, st_);

        // ---------------- loss + LM head forward / backward in row chunks (grpo.hpp:254-272)
        SGB_CUDA(cudaMemsetAsync(p.dlnf, 0, static_cast<size_t>(R) * d * 4, st_));
        for (int r0 = 0; r0 < R; r0 += p.lc) {
            const int rc = std::min(p.lc, R - r0);
            GemmAct af;
            af.init(p.fhat_b + static_cast<size_t>(r0) * d, rc, d);
            GemmEpi e;
            e.kind = kEpiF32;
            e.f32 = p.logits;
            e.ld = V;
            gemm(lm_head_, af, rc, e, kClsLmHead, 4.0);
            launch_ce(p.logits, rc, V, p.next + r0, 0.0, p.dlog, p.loss_row + r0, st_, p.rscale + r0);
            // d_lnf = dlogits . lm_head^T (tinylm.hpp:845-846)
            e = GemmEpi{};
            e.kind = kEpiResid;
            e.f32 = p.dlnf + static_cast<size_t>(r0) * d;
            e.ld = d;
            gemm(p.lm_ref, p.act_dlog, rc, e, kClsLmHead, 8.0);
            // dW_lm[d][V] += lnf_y^T . dlogits (tinylm.hpp:843-844)
            const int rcp = pad8(rc);
            launch_transpose_bf16(p.dlog, rc, V, V, p.tA, rcp, st_);
            launch_transpose_bf16(p.fhat_b + static_cast<size_t>(r0) * d, rc, d, d, p.tB, rcp, st_);
            wgrad(p.tA, V, p.tB, d, rcp, p.grad + tlay_.lm_head, V);
        }
        {
            std::vector<double> lr(R);
            SGB_CUDA(cudaMemcpyAsync(lr.data(), p.loss_row, R * 8, cudaMemcpyDeviceToHost, st_));
            SGB_CUDA(cudaStreamSynchronize(st_));
            for (int r = 0; r < R; ++r) terms.loss += lr[r];
        }

        // ---------------- backward (tinylm.hpp:847-866, 720-800)
        launch_ln_bwd(p.xfin, lnf_g_, p.muf, p.rsf, p.dlnf, nullptr, R, d, p.dx, p.dgb, st_);
        launch_colsum_add(p.dgb, R, 2 * d, p.grad + tlay_.lnf_g, st_);
        for (int l = Ln - 1; l >= 0; --l) {
            Pol::Layer& a = p.L[l];
            const LayerDev& W = tL_[l];
            const auto& lo = tlay_.layers[l];
            const Pol::Refs& rf = p.refs[l];
            // MLP: dW2 += hg^T dx ; d_hg = dx W2^T ; gelu' ; dW1 += a2^T dfch ; d_a2 = dfch W1^T
            launch_transpose_bf16(p.dx, R, d, d, p.tA, Rp, st_);
            launch_transpose_bf16(a.hg, R, F, F, p.tB, Rp, st_);
            wgrad(p.tA, d, p.tB, F, Rp, p.grad + lo.w2, d);
            launch_f32_to_bf16(p.dx, static_cast<size_t>(R) * d, p.dx_b, st_);
            GemmEpi e;
            e.kind = kEpiF32;
            e.f32 = p.dhg;
            e.ld = F;
            gemm(rf.w2, p.act_dx, R, e, kClsGemm, 4.0);
            launch_gelu_bwd(a.fch, p.dhg, static_cast<size_t>(R) * F, p.dfch_b, st_);
            launch_transpose_bf16(p.dfch_b, R, F, F, p.tA, Rp, st_);
            launch_transpose_bf16(a.a2, R, d, d, p.tB, Rp, st_);
            wgrad(p.tA, F, p.tB, d, Rp, p.grad + lo.w1, F);
            e = GemmEpi{};
            e.kind = kEpiF32;
            e.f32 = p.da;
            e.ld = d;
            gemm(rf.w1, p.act_dfch, R, e, kClsGemm, 4.0);
            launch_ln_bwd(a.xmid, W.ln2_g, a.mu2, a.rs2, p.da, p.dx, R, d, p.dxmid, p.dgb, st_);
            launch_colsum_add(p.dgb, R, 2 * d, p.grad + lo.ln2_g, st_);
            // attention: dWo += ctx^T dxmid ; dctx = dxmid Wo^T ; attention bwd ; dWq/k/v ; d_a1
            launch_transpose_bf16(p.dxmid, R, d, d, p.tA, Rp, st_);
            launch_transpose_bf16(a.ctxb, R, d, d, p.tB, Rp, st_);
            wgrad(p.tA, d, p.tB, d, Rp, p.grad + lo.wo, d);
            launch_f32_to_bf16(p.dxmid, static_cast<size_t>(R) * d, p.dxmid_b, st_);
            e = GemmEpi{};
            e.kind = kEpiF32;
            e.f32 = p.dctx;
            e.ld = d;
            gemm(rf.wo, p.act_dxmid, R, e, kClsGemm, 4.0);
            launch_train_attn_bwd(a.qkv, a.ctx, p.dctx, a.lse, p.seq_first, p.seq_last, p.tiles, n_tiles, R, d, H, p.Drow,
                                  p.dqkv, st_);
            launch_transpose_bf16(a.a1, R, d, d, p.tB, Rp, st_);
            const size_t qkv_off[3] = {lo.wq, lo.wk, lo.wv};
            for (int k = 0; k < 3; ++k) {
                launch_transpose_bf16(p.dqkv + static_cast<size_t>(k) * d, R, d, 3 * d, p.tA, Rp, st_);
                wgrad(p.tA, d, p.tB, d, Rp, p.grad + qkv_off[k], d);
            }
            launch_f32_to_bf16(p.dqkv, static_cast<size_t>(R) * 3 * d, p.dqkv_b, st_);
            e = GemmEpi{};
            e.kind = kEpiF32;
            e.f32 = p.da;
            e.ld = d;
            gemm(rf.wqkv, p.act_dqkv, R, e, kClsGemm, 4.0);
            launch_ln_bwd(a.x_in, W.ln1_g, a.mu1, a.rs1, p.da, p.dxmid, R, d, p.dx, p.dgb, st_);
            launch_colsum_add(p.dgb, R, 2 * d, p.grad + lo.ln1_g, st_);
        }
        // embeddings (tinylm.hpp:857-865): rows grouped by token id / by position (CSR)
        for (int which = 0; which < 2; ++which) {
            const std::vector<int>& ids = which ? pos : tok;
            std::vector<int> order(R);
            for (int r = 0; r < R; ++r) order[r] = r;
            std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return ids[x] < ids[y]; });
            std::vector<int> key, ptr{0};
            for (int j = 0; j < R; ++j) {
                if (j == 0 || ids[order[j]] != ids[order[j - 1]]) {
                    if (j) ptr.push_back(j);
                    key.push_back(ids[order[j]]);
                }
            }
            ptr.push_back(R);
            int* dk = p.csr;
            int* dp = p.csr + R;
            int* dr = p.csr + 2 * R + 1;
            SGB_CUDA(cudaMemcpyAsync(dk, key.data(), key.size() * 4, cudaMemcpyHostToDevice, st_));
            SGB_CUDA(cudaMemcpyAsync(dp, ptr.data(), ptr.size() * 4, cudaMemcpyHostToDevice, st_));
            SGB_CUDA(cudaMemcpyAsync(dr, order.data(), R * 4, cudaMemcpyHostToDevice, st_));
            launch_embed_grad(dk, dp, dr, static_cast<int>(key.size()), d, p.dx,
                              p.grad + (which ? tlay_.pos_emb : tlay_.tok_emb), st_);
            SGB_CUDA(cudaStreamSynchronize(st_));  // the host tables are reused
        }
        count(50 * Ln + 20);
    }
    if (A.grad_hook) A.grad_hook(p.grad, tlay_.total, st_, A.hook_ctx);
    if (A.grad_out) SGB_CUDA(cudaMemcpyAsync(A.grad_out, p.grad, tlay_.total * 4, cudaMemcpyDeviceToHost, st_));
    if (A.apply_step) {
        ++p.adam_t;
        launch_adamw(tmaster_, p.grad, p.m, p.v, tlay_.total, A.lr, A.beta1, A.beta2, A.eps, A.weight_decay, p.adam_t,
                     st_);
        convert_target(tmaster_);          // bf16 inference weights, fp32 embeddings / LN params
        policy_refresh_ref_weights();      // dgrad operands
        if (tr2_.ready) draft_lm_stale_ = true;  // the draft update's frozen LM-head copy
    }
    SGB_CUDA(cudaEventRecord(ev1.e, st_));
    SGB_CUDA(cudaEventSynchronize(ev1.e));
    float ms = 0.f;
    SGB_CUDA(cudaEventElapsedTime(&ms, ev0.e, ev1.e));
    terms.seconds = ms * 1e-3;
    return terms;
}

void Engine::policy_adamw_state(float* m, float* v, long long* t, bool upload) {
    policy_alloc();
    const size_t n = tlay_.total;
    if (upload) {
        if (m) SGB_CUDA(cudaMemcpyAsync(pol_.m, m, n * 4, cudaMemcpyHostToDevice, st_));
        else SGB_CUDA(cudaMemsetAsync(pol_.m, 0, n * 4, st_));
        if (v) SGB_CUDA(cudaMemcpyAsync(pol_.v, v, n * 4, cudaMemcpyHostToDevice, st_));
        else SGB_CUDA(cudaMemsetAsync(pol_.v, 0, n * 4, st_));
        pol_.adam_t = t ? *t : 0;
    } else {
        if (m) SGB_CUDA(cudaMemcpyAsync(m, pol_.m, n * 4, cudaMemcpyDeviceToHost, st_));
        if (v) SGB_CUDA(cudaMemcpyAsync(v, pol_.v, n * 4, cudaMemcpyDeviceToHost, st_));
        if (t) *t = pol_.adam_t;
    }
    SGB_CUDA(cudaStreamSynchronize(st_));
}

}  // namespace sgb
