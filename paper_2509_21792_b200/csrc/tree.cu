// Speculation-tree, acceptance-walk and KV-commit kernels (one sequence per warp/CTA).
//
//   tree_root_kernel     -- expand_tree_with level 1 (drafttree.cpp:34-57): root = last
//                           committed token, children = top-k of the root draft logits,
//                           confidence = parent * exp(lp) in fp64.
//   tree_frontier_kernel -- drafttree.cpp:58-67: next frontier = top-k of the previous level
//                           by (confidence desc, token asc, index asc), in index order; emits
//                           the batched draft-forward rows for those nodes with their
//                           ancestor K/V chains (scheduler.cpp:169-199).
//   tree_expand_kernel   -- drafttree.cpp:44-56: append top-k children of each frontier node.
//   tree_select_kernel   -- rerank_candidates + build_tree_mask (drafttree.cpp:126-168):
//                           top-n_verify by (confidence desc, index asc), ascending; emits the
//                           verify-forward rows (token, position p+depth, ancestor chain).
//   walk_commit_kernel   -- verify walk (drafttree.cpp:194-213) + commit_tokens
//                           (scheduler.cpp:97-118): EOS / length-cap stop, finish flags.
//   commit_kv_kernel     -- KvCacheT::gather_tail + truncate (tinylm.hpp:245-268): copies the
//                           accepted rows' K/V from the verify scratch into the cache in order
//                           (scratch and cache never alias, so no read-after-write hazard), and
//                           appends their hidden states to the feature rows (scheduler.cpp:230).
#include "common.cuh"
#include "kernels.h"
#include "util.h"

namespace sgb {

namespace {

constexpr int kEos = 1;  // tinylm.hpp:41

__device__ __forceinline__ bool node_better(double ca, int ta, int ia, double cb, int tb, int ib) {
    if (ca != cb) return ca > cb;
    if (ta != tb) return ta < tb;
    return ia < ib;
}

__global__ void tree_root_kernel(int B, const StepSeqDev* __restrict__ steps, SeqStateDev ss, TreeDev tr,
                                 const int* __restrict__ topk_tok, const double* __restrict__ topk_lp, int kk) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B) return;
    const StepSeqDev st = steps[i];
    const size_t base = static_cast<size_t>(st.seq) * tr.tmax;
    tr.tok[base] = ss.tokens[static_cast<size_t>(st.seq) * ss.max_seq + st.p];
    tr.par[base] = -1;
    tr.dep[base] = 0;
    tr.lp[base] = 0.0;
    tr.conf[base] = 1.0;
    tr.fslot[base] = 0;
    int n = 1;
    if (st.k > 0 && st.root_row >= 0) {
        for (int j = 0; j < st.k; ++j) {
            const double l = topk_lp[static_cast<size_t>(st.root_row) * kk + j];
            tr.tok[base + 1 + j] = topk_tok[static_cast<size_t>(st.root_row) * kk + j];
            tr.par[base + 1 + j] = 0;
            tr.dep[base + 1 + j] = 1;
            tr.lp[base + 1 + j] = l;
            tr.conf[base + 1 + j] = tr.static_rank ? ldexp(1.0, -(j + 1)) : 1.0 * exp(l);
        }
        if (tr.qrow) tr.qrow[base] = st.root_row;
        n = 1 + st.k;
        tr.lvl_start[st.seq] = 1;
        tr.lvl_cnt[st.seq] = st.k;
    }
    tr.n_nodes[st.seq] = n;
}

__global__ void tree_frontier_kernel(int B, int level, const StepSeqDev* __restrict__ steps,
                                     const int* __restrict__ drow_off, SeqStateDev ss, TreeDev tr, RowsDev rows,
                                     long long dcache_stride, long long dscratch_base, int d, int qoff) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int lane = threadIdx.x & 31;
    if (i >= B) return;
    const StepSeqDev st = steps[i];
    if (st.l < level || st.k <= 0) return;
    const int s = st.seq;
    const size_t base = static_cast<size_t>(s) * tr.tmax;
    const int start = tr.lvl_start[s], cnt = tr.lvl_cnt[s], k = st.k;
    int running = 0;
    for (int c0 = 0; c0 < cnt; c0 += 32) {
        const int c = c0 + lane;
        bool selected = false;
        if (c < cnt) {
            const int v = start + c;
            const double cv = tr.conf[base + v];
            // static ranking (rejection mode): the sampled tokens must not steer the shape
            const int tv = tr.static_rank ? 0 : tr.tok[base + v];
            int rank = 0;
            for (int u = start; u < start + cnt; ++u)
                rank += node_better(tr.conf[base + u], tr.static_rank ? 0 : tr.tok[base + u], u, cv, tv, v) ? 1 : 0;
            selected = rank < k;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, selected);
        if (selected) {
            const int pos = running + __popc(bal & ((1u << lane) - 1u));
            tr.frontier[s * 16 + pos] = start + c;
        }
        running += __popc(bal);
    }
    __syncwarp();
    if (lane < k) {
        const int j = lane;
        const int node = tr.frontier[s * 16 + j];
        const int fs = 1 + (level - 2) * k + j;
        tr.fslot[base + node] = fs;
        const int row = drow_off[i] + j;
        const int dn = tr.dep[base + node];
        if (qoff >= 0 && tr.qrow) tr.qrow[base + node] = qoff + row;
        rows.tok[row] = tr.tok[base + node];
        rows.pos[row] = st.p + dn;
        const long long own = dscratch_base + static_cast<long long>(s) * tr.ds + fs;
        rows.kv_dst[row] = own;
        rows.ctx_base[row] = static_cast<long long>(s) * dcache_stride;
        rows.ctx_len[row] = st.p;
        long long* ch = rows.chain + static_cast<size_t>(row) * kMaxChain;
        ch[dn - 1] = own;
        for (int a = tr.par[base + node]; a >= 0 && tr.dep[base + a] >= 1; a = tr.par[base + a])
            ch[tr.dep[base + a] - 1] = dscratch_base + static_cast<long long>(s) * tr.ds + tr.fslot[base + a];
        rows.chain_len[row] = dn;
        const int pf = tr.fslot[base + tr.par[base + node]];
        rows.feat_off[row] = (static_cast<long long>(s) * tr.ds + pf) * d;
        rows.out_off[row] = (static_cast<long long>(s) * tr.ds + fs) * d;
    }
}

__global__ void tree_expand_kernel(int B, int level, const StepSeqDev* __restrict__ steps,
                                   const int* __restrict__ drow_off, TreeDev tr, const int* __restrict__ topk_tok,
                                   const double* __restrict__ topk_lp) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B) return;
    const StepSeqDev st = steps[i];
    if (st.l < level || st.k <= 0) return;
    const int s = st.seq, k = st.k;
    const size_t base = static_cast<size_t>(s) * tr.tmax;
    int n = tr.n_nodes[s];
    const int start = n;
    for (int j = 0; j < k; ++j) {
        const int parent = tr.frontier[s * 16 + j];
        const double pc = tr.conf[base + parent];
        const int row = drow_off[i] + j;
        for (int c = 0; c < k; ++c) {
            const double l = topk_lp[static_cast<size_t>(row) * k + c];
            tr.tok[base + n] = topk_tok[static_cast<size_t>(row) * k + c];
            tr.par[base + n] = parent;
            tr.dep[base + n] = level;
            tr.lp[base + n] = l;
            tr.conf[base + n] = tr.static_rank ? ldexp(pc, -(c + 1)) : pc * exp(l);
            ++n;
        }
    }
    tr.lvl_start[s] = start;
    tr.lvl_cnt[s] = k * k;
    tr.n_nodes[s] = n;
}

constexpr int kSelT = 256;
constexpr int kTmaxCap = 1024;

__global__ void __launch_bounds__(kSelT)
    tree_select_kernel(int B, const StepSeqDev* __restrict__ steps, SeqStateDev ss, TreeDev tr, RowsDev rows,
                       long long tcache_stride, long long tscratch_base, unsigned char* mask_dbg, int* err) {
    pdl_wait();
    pdl_trigger();
    __shared__ double sconf[kTmaxCap];
    __shared__ int spar[kTmaxCap], sdep[kTmaxCap], ssel[kTmaxCap], spos[kTmaxCap];
    const int i = blockIdx.x;
    const StepSeqDev st = steps[i];
    const int s = st.seq;
    const size_t base = static_cast<size_t>(s) * tr.tmax;
    const int n = tr.n_nodes[s];
    const int N = st.nsel;
    for (int v = threadIdx.x; v < n; v += kSelT) {
        sconf[v] = tr.conf[base + v];
        spar[v] = tr.par[base + v];
        sdep[v] = tr.dep[base + v];
    }
    __syncthreads();
    for (int v = threadIdx.x; v < n; v += kSelT) {
        const double cv = sconf[v];
        int rank = 0;
        for (int u = 0; u < n; ++u) rank += (sconf[u] > cv || (sconf[u] == cv && u < v)) ? 1 : 0;
        ssel[v] = rank < N ? 1 : 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int c = 0;
        for (int v = 0; v < n; ++v) spos[v] = ssel[v] ? c++ : -1;
    }
    __syncthreads();
    for (int v = threadIdx.x; v < n; v += kSelT)
        if (spos[v] >= 0) tr.sel[base + spos[v]] = v;
    __syncthreads();
    for (int r = threadIdx.x; r < N; r += kSelT) {
        const int v = tr.sel[base + r];
        const int row = st.vrow_off + r;
        const int dv = sdep[v];
        rows.tok[row] = tr.tok[base + v];
        rows.pos[row] = st.p + dv;
        rows.kv_dst[row] = tscratch_base + row;
        rows.ctx_base[row] = static_cast<long long>(s) * tcache_stride;
        rows.ctx_len[row] = st.p;
        rows.pre_base[row] = st.pre_base;
        rows.pre_len[row] = min(st.pre_len, st.p);
        long long* ch = rows.chain + static_cast<size_t>(row) * kMaxChain;
        for (int a = v; a >= 0; a = spar[a]) {
            const int pa = spos[a];
            if (pa < 0) {
                atomicOr(err, 8);  // closure violation (drafttree.cpp:160)
                break;
            }
            ch[sdep[a]] = tscratch_base + st.vrow_off + pa;
            if (mask_dbg) mask_dbg[static_cast<size_t>(r) * N + pa] = 1;
        }
        rows.chain_len[row] = dv + 1;
        rows.key_pos[row] = st.p + dv + 1;
        rows.seed[row] = ss.seed[s];
        rows.par_row[row] = dv == 0 ? -1 : spos[spar[v]];
    }
}

__global__ void walk_commit_kernel(int B, const StepSeqDev* __restrict__ steps, SeqStateDev ss, TreeDev tr,
                                   RowsDev rows, const int* __restrict__ emitted, int* __restrict__ acc_rows,
                                   int* __restrict__ result) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B) return;
    const StepSeqDev st = steps[i];
    const int off = st.vrow_off, N = st.nsel;
    int acc_tok[kMaxChain + 1];
    int nacc = 0, cur = 0;
    acc_rows[i * kMaxChain] = 0;
    for (;;) {
        const int want = emitted[off + cur];
        int nxt = -1;
        for (int r = cur + 1; r < N; ++r)
            if (rows.par_row[off + r] == cur && rows.tok[off + r] == want) {
                nxt = r;
                break;
            }
        if (nxt < 0 || nacc + 1 >= kMaxChain) break;
        acc_tok[nacc++] = want;
        acc_rows[i * kMaxChain + nacc] = nxt;
        cur = nxt;
    }
    acc_tok[nacc++] = emitted[off + cur];
    commit_tokens_dev(st, ss, acc_tok, nacc, result + 2 * i);
}

__global__ void commit_kv_kernel(const StepSeqDev* __restrict__ steps, const int* __restrict__ acc_rows,
                                 const int* __restrict__ result, int d, __nv_bfloat16* __restrict__ K,
                                 __nv_bfloat16* __restrict__ V, long long layer_stride, long long tcache_stride,
                                 long long tscratch_base, const float* __restrict__ hidden, float* __restrict__ feats,
                                 int max_seq) {
    pdl_wait();
    pdl_trigger();
    // one CTA per (sequence, layer) walks the accepted rows (1 in AR steps)
    const int i = blockIdx.x, layer = blockIdx.y;
    const int n_acc = result[2 * i];
    const StepSeqDev st = steps[i];
    const size_t lo = static_cast<size_t>(layer) * layer_stride;
    for (int j = 0; j < n_acc; ++j) {
        const int vr = st.vrow_off + acc_rows[i * kMaxChain + j];
        const long long src = tscratch_base + vr;
        const long long dst = static_cast<long long>(st.seq) * tcache_stride + st.p + j;
        const uint4* ks = reinterpret_cast<const uint4*>(K + lo + src * d);
        const uint4* vs = reinterpret_cast<const uint4*>(V + lo + src * d);
        uint4* kd = reinterpret_cast<uint4*>(K + lo + dst * d);
        uint4* vd = reinterpret_cast<uint4*>(V + lo + dst * d);
        for (int e = threadIdx.x; e < d / 8; e += blockDim.x) {
            kd[e] = ks[e];
            vd[e] = vs[e];
        }
        if (layer == 0) {
            const float* h = hidden + static_cast<size_t>(vr) * d;
            float* f = feats + (static_cast<size_t>(st.seq) * max_seq + st.p + j) * d;
            for (int e = threadIdx.x; e < d; e += blockDim.x) f[e] = h[e];
        }
    }
}

__global__ void copy_rows_f32_kernel(const float* __restrict__ src, const int* __restrict__ src_row,
                                     const long long* __restrict__ dst_off, int d, float* __restrict__ dst) {
    pdl_wait();
    pdl_trigger();
    const int r = blockIdx.x;
    const float* s = src + static_cast<size_t>(src_row ? src_row[r] : r) * d;
    float* o = dst + dst_off[r];
    for (int e = threadIdx.x; e < d; e += blockDim.x) o[e] = s[e];
}

__global__ void copy_kv_prefix_kernel(const int* __restrict__ src_seq, const int* __restrict__ dst_seq,
                                      const int* __restrict__ plen, int d, __nv_bfloat16* __restrict__ K,
                                      __nv_bfloat16* __restrict__ V, long long layer_stride, long long seq_stride) {
    pdl_wait();
    pdl_trigger();
    const int pr = blockIdx.x, layer = blockIdx.y, t = blockIdx.z;
    if (t >= plen[pr]) return;
    const size_t lo = static_cast<size_t>(layer) * layer_stride;
    const size_t so = (static_cast<size_t>(src_seq[pr]) * seq_stride + t) * d;
    const size_t dof = (static_cast<size_t>(dst_seq[pr]) * seq_stride + t) * d;
    const uint4* ks = reinterpret_cast<const uint4*>(K + lo + so);
    const uint4* vs = reinterpret_cast<const uint4*>(V + lo + so);
    uint4* kd = reinterpret_cast<uint4*>(K + lo + dof);
    uint4* vd = reinterpret_cast<uint4*>(V + lo + dof);
    for (int e = threadIdx.x; e < d / 8; e += blockDim.x) {
        kd[e] = ks[e];
        vd[e] = vs[e];
    }
}

__global__ void prefill_commit_kernel(int n, const int* __restrict__ seqs, const int* __restrict__ qlen,
                                      const int* __restrict__ len_cap, const int* __restrict__ emitted, SeqStateDev ss) {
    pdl_wait();
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int s = seqs[i], q = qlen[i], t = emitted[i];
    ss.tokens[static_cast<size_t>(s) * ss.max_seq + q] = t;
    ss.len[s] = q + 1;
    const int eos = t == kEos;
    ss.hit_eos[s] = eos;
    ss.finished[s] = (eos || q + 1 >= len_cap[i]) ? 1 : 0;
}

__global__ void gather_tokens_kernel(const int* __restrict__ seq, const int* __restrict__ pos, int R, SeqStateDev ss,
                                     int* __restrict__ out) {
    pdl_wait();
    pdl_trigger();
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < R) out[r] = ss.tokens[static_cast<size_t>(seq[r]) * ss.max_seq + pos[r]];
}

}  // namespace

void launch_tree_root(int B, const StepSeqDev* steps, const SeqStateDev& ss, const TreeDev& tr, const int* topk_tok,
                      const double* topk_lp, int kk, cudaStream_t st) {
    if (B <= 0) return;
    launch_pdl(tree_root_kernel, (B + 127) / 128, 128, 0, st, B, steps, ss, tr, topk_tok, topk_lp, kk);
    SGB_KCHECK();
}

void launch_tree_frontier(int B, int level, const StepSeqDev* steps, const int* drow_off, const SeqStateDev& ss,
                          const TreeDev& tr, const RowsDev& rows, long long dcache_stride, long long dscratch_base,
                          int d, cudaStream_t st, int qoff) {
    if (B <= 0) return;
    launch_pdl(tree_frontier_kernel, (B + 3) / 4, 128, 0, st, B, level, steps, drow_off, ss, tr, rows, dcache_stride,
                                                      dscratch_base, d, qoff);
    SGB_KCHECK();
}

void launch_tree_expand(int B, int level, const StepSeqDev* steps, const int* drow_off, const TreeDev& tr,
                        const int* topk_tok, const double* topk_lp, cudaStream_t st) {
    if (B <= 0) return;
    launch_pdl(tree_expand_kernel, (B + 127) / 128, 128, 0, st, B, level, steps, drow_off, tr, topk_tok, topk_lp);
    SGB_KCHECK();
}

void launch_tree_select(int B, const StepSeqDev* steps, const SeqStateDev& ss, const TreeDev& tr, const RowsDev& rows,
                        long long tcache_stride, long long tscratch_base, unsigned char* mask_dbg, int* err,
                        cudaStream_t st) {
    if (B <= 0) return;
    if (tr.tmax > kTmaxCap) throw std::invalid_argument("tree capacity exceeds 1024 nodes");
    launch_pdl(tree_select_kernel, B, kSelT, 0, st, B, steps, ss, tr, rows, tcache_stride, tscratch_base, mask_dbg, err);
    SGB_KCHECK();
}

void launch_walk_commit(int B, const StepSeqDev* steps, const SeqStateDev& ss, const TreeDev& tr, const RowsDev& rows,
                        const int* emitted, int* acc_rows, int* result, cudaStream_t st) {
    if (B <= 0) return;
    launch_pdl(walk_commit_kernel, (B + 127) / 128, 128, 0, st, B, steps, ss, tr, rows, emitted, acc_rows, result);
    SGB_KCHECK();
}

void launch_commit_kv(int B, const StepSeqDev* steps, const int* acc_rows, const int* result, int layers, int d,
                      __nv_bfloat16* K, __nv_bfloat16* V, long long layer_stride, long long tcache_stride,
                      long long tscratch_base, const float* hidden, float* feats, int max_seq, cudaStream_t st) {
    if (B <= 0) return;
    dim3 grid(B, layers);
    launch_pdl(commit_kv_kernel, grid, 128, 0, st, steps, acc_rows, result, d, K, V, layer_stride, tcache_stride,
                                           tscratch_base, hidden, feats, max_seq);
    SGB_KCHECK();
}

void launch_copy_rows_f32(const float* src, const int* src_row, const long long* dst_off, int R, int d, float* dst,
                          cudaStream_t st) {
    if (R <= 0) return;
    launch_pdl(copy_rows_f32_kernel, R, 256, 0, st, src, src_row, dst_off, d, dst);
    SGB_KCHECK();
}

void launch_copy_kv_prefix(const int* src_seq, const int* dst_seq, const int* plen, int n, int max_plen, int layers,
                           int d, __nv_bfloat16* K, __nv_bfloat16* V, long long layer_stride, long long seq_stride,
                           cudaStream_t st) {
    if (n <= 0 || max_plen <= 0) return;
    launch_pdl(copy_kv_prefix_kernel, dim3(n, layers, max_plen), 128, 0, st, src_seq, dst_seq, plen, d, K, V, layer_stride,
                                                                     seq_stride);
    SGB_KCHECK();
}

void launch_prefill_commit(int n, const int* seqs, const int* qlen, const int* len_cap, const int* emitted,
                           const SeqStateDev& ss, cudaStream_t st) {
    if (n <= 0) return;
    launch_pdl(prefill_commit_kernel, (n + 127) / 128, 128, 0, st, n, seqs, qlen, len_cap, emitted, ss);
    SGB_KCHECK();
}

void launch_gather_tokens(const int* seq, const int* pos, int R, const SeqStateDev& ss, int* out, cudaStream_t st) {
    if (R <= 0) return;
    launch_pdl(gather_tokens_kernel, (R + 127) / 128, 128, 0, st, seq, pos, R, ss, out);
    SGB_KCHECK();
}

}  // namespace sgb
