// Speculative REJECTION SAMPLING -- the `acceptance = 1` rollout mode (north star item 3,
// BASELINE configs[4] "rejection-sampling verify at T=1.0").
//
// The reference only has keyed strict-match acceptance (verify, drafttree.cpp:170-222): the
// target emits a keyed sample at every selected node and a child is accepted if it carries that
// token. With deterministic top-k children that is already lossless, and its acceptance rate is
// the target mass of the candidates -- at T = 1 over a 128k-152k vocabulary that mass is tiny
// however good the draft is. Standard speculative sampling instead SAMPLES the candidates from
// the draft distribution q and accepts candidate x with probability min(1, p(x) / q(x)); with
// several candidates per node it is the multi-round form (SpecInfer): after a rejection the
// target distribution is replaced by the residual norm(max(p - q, 0)) and the next candidate
// is tried; when all are rejected the bonus token is drawn from the final residual. Each
// emitted token is then distributed exactly as p, and a candidate is accepted with probability
// 1 - TV(p, q) per round, so a draft that has learned q ~ p is accepted almost always.
//
// Losslessness needs every node's verified children to be a prefix of an i.i.d. sequence from
// q that was chosen without looking at the sampled values, so in this mode the tree shape is
// static: children carry the exact dyadic confidences conf(parent) * 2^-(j+1) and every
// frontier / rerank tie is broken by node index (tree.cu, TreeDev::static_rank). The expansion
// and verify machinery (batched draft levels, tree-masked verify forward, KV commit) is the
// same as the strict-match mode's.
//
// Keys (no reference behaviour to match; the parity mode is strict match): child c of a node
// whose children sit at position p is mix_key(mix_key(mix_key(seq_seed, p), 0xD5A0 + f), c),
// f = the node's frontier index; the acceptance uniform of child j is
// mix_key(mix_key(seq_seed, p), 0xACC0 + j); the residual bonus uses 0xB0B0. A node with no
// selected children emits the keyed sample_token draw of its row (emit kernels), so steps
// without speculation are bit-identical to the strict-match mode.
#include <cfloat>

#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.h"
#include "util.h"

namespace cg = cooperative_groups;

namespace sgb {

namespace {

constexpr int kRT = 512;  // threads per row CTA

// a row's terms exp((l - m) / T) in fp32 (summed in fp64): any fixed function defines q / p
// exactly as long as the same one evaluates the sampling CDF and the acceptance ratios; fp32
// exp is ~10x cheaper than fp64 on the full-vocabulary passes of the walk
SGB_DEV double term(float l, double m, double temperature) {
    return static_cast<double>(__expf(__fdividef(l - static_cast<float>(m), static_cast<float>(temperature))));
}

// block max of a float row
SGB_DEV float block_max(const float* L, int V, float* red) {
    float m = -INFINITY;
    for (int i = threadIdx.x; i < V; i += blockDim.x) m = fmaxf(m, L[i]);
    m = warp_max(m);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    float r = red[0];
    for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) r = fmaxf(r, red[w]);
    __syncthreads();
    return r;
}

SGB_DEV double block_sum(double v, double* red) {
    v = warp_sum_d(v);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) r += red[w];
    __syncthreads();
    return r;
}

struct RowStat {
    double m, z;
};

SGB_DEV RowStat row_stat(const float* L, int V, double temperature, float* redf, double* redd) {
    const double m = static_cast<double>(block_max(L, V, redf));
    double s = 0.0;
    for (int i = threadIdx.x; i < V; i += blockDim.x) s += term(L[i], m, temperature);
    return RowStat{m, block_sum(s, redd)};
}

// ---- cluster form of the walk (thread-block clusters of kCL CTAs per sequence, DSMEM reductions)
//
// A node's passes are full-vocabulary sweeps; one CTA per sequence streams them through one SM
// (a 152k-logit row pair at ~150 GB/s per SM), so at low concurrency the walk took ~1.5 ms per
// step. Here a cluster of kCL CTAs splits the vocabulary, and every sum is a cluster reduction
// over distributed shared memory (fixed rank order: all CTAs get the same bits and take the same
// decisions). The residual needs no buffer: after j rejections at a node it is
// max(p - c_j q, 0) / W(c_j) with c_0 = 0, c_{j+1} = c_j + W(c_j), W(c) = sum max(p - c q, 0) --
// the same distribution as norm(max(r - q, 0)) applied j times, recomputed on the fly.
constexpr int kCL = 8;

SGB_DEV double cluster_sum(cg::cluster_group& cl, double v_block, double* xch) {
    if (threadIdx.x == 0) *xch = v_block;
    cl.sync();
    double s = 0.0;
    for (int r = 0; r < kCL; ++r) s += *cl.map_shared_rank(xch, r);
    cl.sync();
    return s;
}

struct Slice {
    int lo, hi;
};
SGB_DEV Slice vocab_slice(int V, int rank) {
    const int per = (V + kCL - 1) / kCL;
    const int lo = min(V, rank * per);
    return Slice{lo, min(V, lo + per)};
}

// Block-wide exclusive scan of per-thread doubles (shuffle scan per warp, then over the warp
// totals): pre[t] = sum of v over threads < t, pre[blockDim.x] = the block total. The owner test
// of a draw compares against pre[t] and pre[t + 1] only, so neighbouring intervals share their
// bounds exactly and every u in [0, total) has exactly one owner. wsum: shared [32].
SGB_DEV void block_excl_scan(double v, double* pre, double* wsum) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    double ex = __shfl_up_sync(0xffffffffu, x, 1);
    if (lane == 0) ex = 0.0;
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        double t = lane < nw ? wsum[lane] : 0.0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double y = __shfl_up_sync(0xffffffffu, t, o);
            if (lane >= o) t += y;
        }
        if (lane < nw) wsum[lane] = t;  // inclusive warp prefix
    }
    __syncthreads();
    pre[threadIdx.x] = (w > 0 ? wsum[w - 1] : 0.0) + ex;
    if (threadIdx.x == 0) pre[blockDim.x] = wsum[nw - 1];
    __syncthreads();
}

// Inverse CDF over the vocabulary in index order, split over the cluster: rank r owns the slice
// vocab_slice(V, r), thread t of it the contiguous segment [lo, hi). After setup every thread
// knows its interval [before + pre[t], before + pre[t + 1]) of the cluster-wide CDF (the same
// floating-point expressions on both sides of every boundary), so a draw u is resolved by its
// unique owner alone -- k draws run in parallel with no further synchronisation. u >= total
// (rounding only) goes to the last thread with mass, which returns its last positive index.
struct ClusterCdf {
    int lo, hi;
    double before, total;
    bool last_owner;
};

template <class W>
SGB_DEV ClusterCdf cluster_cdf(cg::cluster_group& cl, W w, Slice sl, double* pre, double* wsum, double* xch,
                               int* xlast) {
    const int T = blockDim.x, t = threadIdx.x;
    const int n = sl.hi - sl.lo;
    const int seg = (n + T - 1) / T;
    ClusterCdf c;
    c.lo = sl.lo + min(n, t * seg);
    c.hi = min(sl.hi, c.lo + seg);
    double s = 0.0;
    for (int i = c.lo; i < c.hi; ++i) s += w(i);
    if (t == 0) *xlast = -1;
    __syncthreads();
    if (s > 0.0) atomicMax(xlast, t);
    block_excl_scan(s, pre, wsum);  // (syncs: xlast complete)
    if (t == 0) *xch = pre[T];
    cl.sync();
    const int me = static_cast<int>(cl.block_rank());
    double before = 0.0, total = 0.0;
    int last_rank = -1;
    for (int r = 0; r < kCL; ++r) {
        const double x = *cl.map_shared_rank(xch, r);
        if (r == me) before = total;
        total += x;
        if (x > 0.0) last_rank = r;
    }
    c.before = before;
    c.total = total;
    c.last_owner = (me == last_rank && t == *xlast);
    return c;
}

// the owner's walk; -1 if this thread does not own u
template <class W>
SGB_DEV int cdf_owner_draw(const ClusterCdf& c, W w, const double* pre, double u) {
    const int t = threadIdx.x;
    const double lo = c.before + pre[t], hi = c.before + pre[t + 1];
    const bool mine = (lo <= u && u < hi) || (!(u < c.total) && c.last_owner);
    if (!mine) return -1;
    double acc = lo;
    int last = c.lo;
    for (int i = c.lo; i < c.hi; ++i) {
        const double x = w(i);
        if (x > 0.0) last = i;
        acc += x;
        if (u < acc) return i;
    }
    return last;
}

// one draw broadcast to the whole cluster. xtok: this CTA's exchange slot (shared memory).
template <class W>
SGB_DEV int cluster_draw(cg::cluster_group& cl, W w, Slice sl, double u01, double* pre, double* wsum, double* xch,
                         int* xlast, int* xtok) {
    if (threadIdx.x == 0) *xtok = 0;  // (total == 0 cannot happen: p and the residuals have mass)
    const ClusterCdf c = cluster_cdf(cl, w, sl, pre, wsum, xch, xlast);
    const int tok = cdf_owner_draw(c, w, pre, u01 * c.total);
    if (tok >= 0)
        for (int r = 0; r < kCL; ++r) *cl.map_shared_rank(xtok, r) = tok;
    cl.sync();
    const int res = *xtok;
    cl.sync();  // xch / xtok are reused by the next exchange
    return res;
}

SGB_DEV float cluster_max(cg::cluster_group& cl, float v_block, float* xf) {
    if (threadIdx.x == 0) *xf = v_block;
    cl.sync();
    float m = -INFINITY;
    for (int r = 0; r < kCL; ++r) m = fmaxf(m, *cl.map_shared_rank(xf, r));
    cl.sync();
    return m;
}

// One node of the multi-round walk on a cluster. P / Q: target / draft logit rows; cand[n]: the
// node's verified children (a prefix of its i.i.d. samples). Returns the accepted candidate's
// index, or -1 with *bonus drawn from the final residual.
struct ClusterSmem {
    double pre[kRT + 1];
    double wsum[32];
    double redd[kRT / 32];
    double xch;
    float redf[kRT / 32];
    float xf;
    int xlast, xtok;
};

// The node's p and q terms over this CTA's slice are staged once in shared memory (stage[0..n) =
// p terms, stage[n..2n) = q terms, fp32 exactly as term() returns them), so the residual passes
// and the bonus CDF read shared memory; a candidate outside the slice recomputes the same term.
SGB_DEV int mss_node_cluster(cg::cluster_group& cl, const float* P, double pm, const float* Q, RowStat qs,
                             const int* cand, int n, int V, double temperature, uint64_t key, ClusterSmem& sm,
                             float* stage, int* bonus) {
    const Slice sl = vocab_slice(V, static_cast<int>(cl.block_rank()));
    const int ns = sl.hi - sl.lo;
    float* tp = stage;
    float* tq = stage + ns;
    double zs = 0.0;
    for (int i = threadIdx.x; i < ns; i += blockDim.x) {
        const double a = term(P[sl.lo + i], pm, temperature);
        tp[i] = static_cast<float>(a);
        tq[i] = static_cast<float>(term(Q[sl.lo + i], qs.m, temperature));
        zs += a;
    }
    const double zp = cluster_sum(cl, block_sum(zs, sm.redd), &sm.xch);  // (block_sum syncs: stage complete)
    const double izp = 1.0 / zp, iqz = 1.0 / qs.z;
    auto pn = [&](int i) { return static_cast<double>(tp[i - sl.lo]) * izp; };
    auto qn = [&](int i) { return static_cast<double>(tq[i - sl.lo]) * iqz; };
    double c = 0.0, wc = 1.0;  // residual max(p - c q, 0) / wc
    for (int j = 0; j < n; ++j) {
        const int x = cand[j];
        const double qx = term(Q[x], qs.m, temperature) * iqz;
        const double px = term(P[x], pm, temperature) * izp;
        const double rx = fmax(px - c * qx, 0.0) / wc;
        const double u = rng_first_uniform(mix_key(key, 0xACC0u + j));
        if (u * qx < rx) return j;  // accept with probability min(1, r(x) / q(x))
        c += wc;
        double ws = 0.0;
        for (int i = sl.lo + threadIdx.x; i < sl.hi; i += blockDim.x) ws += fmax(pn(i) - c * qn(i), 0.0);
        wc = cluster_sum(cl, block_sum(ws, sm.redd), &sm.xch);
        if (!(wc > 0.0)) {  // p == c q on the support (floating-point residue): back to p
            c = 0.0;
            wc = 1.0;
        }
    }
    const double ub = rng_first_uniform(mix_key(key, 0xB0B0u));
    if (c == 0.0)
        *bonus = cluster_draw(cl, pn, sl, ub, sm.pre, sm.wsum, &sm.xch, &sm.xlast, &sm.xtok);
    else
        *bonus = cluster_draw(cl, [&](int i) { return fmax(pn(i) - c * qn(i), 0.0); }, sl, ub, sm.pre, sm.wsum,
                              &sm.xch, &sm.xlast, &sm.xtok);
    __syncthreads();  // the stage is rewritten by the next node
    return -1;
}

// dynamic shared memory of the walk kernels: the p / q term stage of one vocabulary slice
inline size_t walk_stage_bytes(int V) {
    const size_t b = 2 * sizeof(float) * static_cast<size_t>((V + kCL - 1) / kCL);
    if (b > (200u << 10)) throw std::invalid_argument("rejection sampling: vocabulary above 200k is unsupported");
    return b;
}

// K children per row, i.i.d. from q = softmax(row / T): one cluster per row (vocabulary split
// over kCL CTAs), one CDF pass, then every draw is resolved by its owning thread in parallel.
// qstat[r] = (m, z) with z the cluster total of the same terms the draws use.
__global__ void __launch_bounds__(kRT) sample_children_kernel(const float* __restrict__ q, int V, int k,
                                                              double temperature,
                                                              const unsigned long long* __restrict__ keys,
                                                              int* __restrict__ out_tok, double* __restrict__ out_lp,
                                                              double* __restrict__ qstat) {
    pdl_wait();
    pdl_trigger();
    cg::cluster_group cl = cg::this_cluster();
    __shared__ ClusterSmem sm;
    const int r = blockIdx.x / kCL;
    const float* Q = q + static_cast<size_t>(r) * V;
    const Slice sl = vocab_slice(V, static_cast<int>(cl.block_rank()));
    float mloc = -INFINITY;
    for (int i = sl.lo + threadIdx.x; i < sl.hi; i += blockDim.x) mloc = fmaxf(mloc, Q[i]);
    mloc = warp_max(mloc);
    if ((threadIdx.x & 31) == 0) sm.redf[threadIdx.x >> 5] = mloc;
    __syncthreads();
    float mb = sm.redf[0];
    for (int w = 1; w < kRT / 32; ++w) mb = fmaxf(mb, sm.redf[w]);
    const double m = static_cast<double>(cluster_max(cl, mb, &sm.xf));
    auto wq = [&](int i) { return term(Q[i], m, temperature); };
    const ClusterCdf c = cluster_cdf(cl, wq, sl, sm.pre, sm.wsum, &sm.xch, &sm.xlast);
    if (cl.block_rank() == 0 && threadIdx.x == 0) {
        qstat[2 * r] = m;
        qstat[2 * r + 1] = c.total;
    }
    for (int j = 0; j < k; ++j) {
        const double u = rng_first_uniform(mix_key(keys[r], static_cast<uint64_t>(j))) * c.total;
        const int tok = cdf_owner_draw(c, wq, sm.pre, u);
        if (tok >= 0) {
            out_tok[static_cast<size_t>(r) * k + j] = tok;
            out_lp[static_cast<size_t>(r) * k + j] = log(wq(tok) / c.total);
        }
    }
    cl.sync();  // the slice totals in shared memory are read by the other ranks until here
}

// one cluster of kCL CTAs per live sequence: the multi-round walk from the root along accepted
// children (every CTA takes the same decisions; rank 0 writes the results)
__global__ void __launch_bounds__(kRT) walk_reject_kernel(int B, const StepSeqDev* __restrict__ steps, SeqStateDev ss,
                                                          TreeDev tr, RowsDev rows, const int* __restrict__ emitted,
                                                          const float* __restrict__ logits,
                                                          const float* __restrict__ rowmax,
                                                          const float* __restrict__ qbuf,
                                                          const double* __restrict__ qstat, int V, double temperature,
                                                          int* __restrict__ acc_rows, int* __restrict__ result) {
    pdl_wait();
    pdl_trigger();
    cg::cluster_group cl = cg::this_cluster();
    __shared__ ClusterSmem sm;
    extern __shared__ float stage[];
    __shared__ int sh_n;
    __shared__ int cand_row[16], cand_tok[16];
    __shared__ int acc_tok[kMaxChain + 1];
    const bool lead = cl.block_rank() == 0;
    const int i = blockIdx.x / kCL;
    const StepSeqDev st = steps[i];
    const int s = st.seq, off = st.vrow_off, N = st.nsel;
    const size_t base = static_cast<size_t>(s) * tr.tmax;
    int cur = 0, nacc = 0;
    if (lead && threadIdx.x == 0) acc_rows[i * kMaxChain] = 0;
    for (;;) {
        // the node's verified children, in row order (a prefix of its sampled children)
        if (threadIdx.x == 0) {
            int n = 0;
            for (int r = cur + 1; r < N && n < 16; ++r)
                if (rows.par_row[off + r] == cur) {
                    cand_row[n] = r;
                    cand_tok[n] = rows.tok[off + r];
                    ++n;
                }
            sh_n = n;
        }
        __syncthreads();
        const int n = sh_n;
        if (n == 0 || nacc + 1 >= kMaxChain) {
            if (threadIdx.x == 0) acc_tok[nacc++] = emitted[off + cur];  // keyed sample_token draw
            break;
        }
        const float* P = logits + static_cast<size_t>(off + cur) * V;
        const double pm = static_cast<double>(rowmax[off + cur]);
        const int node = tr.sel[base + cur];
        const int qr = tr.qrow[base + node];
        const RowStat qs{qstat[2 * qr], qstat[2 * qr + 1]};
        const int depth = tr.dep[base + node];
        const uint64_t key = mix_key(ss.seed[s], static_cast<uint64_t>(st.p + depth + 1));
        int bonus = 0;
        const int j = mss_node_cluster(cl, P, pm, qbuf + static_cast<size_t>(qr) * V, qs, cand_tok, n, V, temperature,
                                       key, sm, stage, &bonus);
        if (j < 0) {
            if (threadIdx.x == 0) acc_tok[nacc++] = bonus;
            break;
        }
        if (threadIdx.x == 0) {
            acc_tok[nacc] = cand_tok[j];
            if (lead) acc_rows[i * kMaxChain + nacc + 1] = cand_row[j];
        }
        ++nacc;
        cur = cand_row[j];
        __syncthreads();
    }
    __syncthreads();
    if (lead && threadIdx.x == 0) commit_tokens_dev(st, ss, acc_tok, nacc, result + 2 * i);
    cl.sync();  // no CTA leaves while its shared memory may still be read
}

__global__ void __launch_bounds__(kRT) debug_spec_kernel(const float* __restrict__ p, const float* __restrict__ q,
                                                         int V, int k, double temperature, unsigned long long seed,
                                                         int* __restrict__ out_tok, int* __restrict__ out_acc) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ ClusterSmem sm;
    extern __shared__ float stage[];
    __shared__ int cand[16];
    const int trial = blockIdx.x / kCL;
    const double pm = static_cast<double>(block_max(p, V, sm.redf));
    const RowStat qs = row_stat(q, V, temperature, sm.redf, sm.redd);
    const uint64_t key = mix_key(seed, static_cast<uint64_t>(trial));
    const Slice sl = vocab_slice(V, static_cast<int>(cl.block_rank()));
    for (int c = 0; c < k; ++c) {
        const double u = rng_first_uniform(mix_key(mix_key(key, 0xD5A0u), static_cast<uint64_t>(c)));
        const int x = cluster_draw(cl, [&](int i) { return term(q[i], qs.m, temperature); }, sl, u, sm.pre, sm.wsum,
                                   &sm.xch, &sm.xlast, &sm.xtok);
        if (threadIdx.x == 0) cand[c] = x;
        __syncthreads();
    }
    int bonus = 0;
    const int j = mss_node_cluster(cl, p, pm, q, qs, cand, k, V, temperature, key, sm, stage, &bonus);
    if (cl.block_rank() == 0 && threadIdx.x == 0) {
        out_tok[trial] = j >= 0 ? cand[j] : bonus;
        out_acc[trial] = j >= 0 ? 1 : 0;
    }
    cl.sync();
}

// grid of kCL-CTA clusters (+ programmatic dependent launch)
template <class... KA, class... A>
void launch_cluster(void (*kern)(KA...), int clusters, size_t smem, bool pdl, cudaStream_t st, A... args) {
    if (smem > 0) SGB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    cudaLaunchConfig_t cfg = {};
    cfg.dynamicSmemBytes = smem;
    cfg.gridDim = dim3(clusters * kCL);
    cfg.blockDim = dim3(kRT);
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kCL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 2 : 1;
    SGB_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KA>(args)...));
}

}  // namespace

void launch_sample_children(const float* q, int R, int V, int k, double temperature, const unsigned long long* keys,
                            int* out_tok, double* out_lp, double* qstat, cudaStream_t st) {
    if (R <= 0) return;
    if (k < 1 || k > 16) throw std::invalid_argument("sample_children: k must be in [1, 16]");
    if (!(temperature > 0)) throw std::invalid_argument("rejection sampling needs temperature > 0");
    launch_cluster(sample_children_kernel, R, 0, true, st, q, V, k, temperature, keys, out_tok, out_lp, qstat);
    SGB_KCHECK();
}

void launch_walk_reject(int B, const StepSeqDev* steps, const SeqStateDev& ss, const TreeDev& tr, const RowsDev& rows,
                        const int* emitted, const float* logits, const float* rowmax, const float* qbuf,
                        const double* qstat, int V, double temperature, float* /*resid*/, int* acc_rows, int* result,
                        cudaStream_t st) {
    if (B <= 0) return;
    launch_cluster(walk_reject_kernel, B, walk_stage_bytes(V), true, st, B, steps, ss, tr, rows, emitted, logits, rowmax, qbuf, qstat, V,
                   temperature, acc_rows, result);
    SGB_KCHECK();
}

void launch_debug_spec_sample(const float* p, const float* q, int V, int k, double temperature, int n_trials,
                              unsigned long long seed, float* /*resid*/, int* out_tok, int* out_acc, cudaStream_t st) {
    if (n_trials <= 0) return;
    if (k < 1 || k > 16) throw std::invalid_argument("debug_spec_sample: k in [1, 16]");
    launch_cluster(debug_spec_kernel, n_trials, walk_stage_bytes(V), false, st, p, q, V, k, temperature, seed, out_tok, out_acc);
    SGB_KCHECK();
}

}  // namespace sgb
