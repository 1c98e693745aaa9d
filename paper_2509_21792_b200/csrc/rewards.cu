// GRPO group rewards and advantages on the device, straight from the rollout's token table.
//
// Reference (src/grpo.cpp):
//   compute_reward (:99-116)          1.0 iff the response's final "=" is followed by the
//                                     decimal digits of a+b (an EOS allowed only as the very
//                                     last token), else 0.0; malformed / > 15 digits -> 0.0
//   standardize_advantages (:121-136) population mean / variance of the group's rewards;
//                                     nullopt (the group is filtered) when sd < eps_var,
//                                     else (r - mean) / sd
//   call site (:352-380)              response = tokens[prompt_len:], sequence s belongs to
//                                     query s / G (generate_dynamic_batch's order)
// Task token ids (include/sgrpo/grpo.hpp:19-21): digit d = 2 + d, '+' = 12, '=' = 13; EOS = 1.
//
// One thread per sequence scans its response; one thread per group reduces in member order
// with every fp64 rounding spelled out, matching the reference binary's operation sequence.
#include "common.cuh"
#include "kernels.h"
#include "util.h"

namespace sgb {

namespace {

constexpr int kDigit0 = 2, kEq = 13, kEosTok = 1;

__global__ void rewards_kernel(int n, const int* __restrict__ tok, long long stride, const int* __restrict__ len,
                               const int* __restrict__ plen, const long long* __restrict__ answer, int g,
                               double* __restrict__ rewards) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const int* t = tok + static_cast<size_t>(s) * stride + plen[s];
    const int rl = len[s] - plen[s];
    int last_eq = -1;
    for (int i = 0; i < rl; ++i)
        if (t[i] == kEq) last_eq = i;
    double r = 0.0;
    if (last_eq >= 0) {
        long long value = 0;
        int digits = 0;
        bool bad = false;
        for (int i = last_eq + 1; i < rl; ++i) {
            const int x = t[i];
            if (x == kEosTok && i + 1 == rl) break;
            if (x < kDigit0 || x >= kDigit0 + 10) {
                bad = true;
                break;
            }
            value = value * 10 + (x - kDigit0);
            if (++digits > 15) {
                bad = true;
                break;
            }
        }
        if (!bad && digits > 0 && value == answer[s / g]) r = 1.0;
    }
    rewards[s] = r;
}

__global__ void advantages_kernel(int n_groups, int g, const double* __restrict__ rewards, double eps_var,
                                  double* __restrict__ adv, int* __restrict__ valid) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n_groups) return;
    const double* r = rewards + static_cast<size_t>(b) * g;
    double mean = 0.0;
    for (int i = 0; i < g; ++i) mean = __dadd_rn(mean, r[i]);
    mean = __ddiv_rn(mean, static_cast<double>(g));
    double var = 0.0;
    // the reference as compiled adds exact squares in order and fuses the odd tail element
    // (vectorised loop + vfmadd231sd remainder, oracle.standardize_advantages)
    for (int i = 0; i < g; ++i) {
        const double dv = __dsub_rn(r[i], mean);
        var = (g % 2 == 1 && i == g - 1) ? __fma_rn(dv, dv, var) : __dadd_rn(var, __dmul_rn(dv, dv));
    }
    var = __ddiv_rn(var, static_cast<double>(g));
    const double sd = __dsqrt_rn(var);
    const bool ok = !(sd < eps_var);
    valid[b] = ok ? 1 : 0;
    for (int i = 0; i < g; ++i) adv[static_cast<size_t>(b) * g + i] = ok ? __ddiv_rn(__dsub_rn(r[i], mean), sd) : 0.0;
}

}  // namespace

void launch_group_advantages(int n_groups, int g, const int* tok, long long stride, const int* len, const int* plen,
                             const long long* answer, double eps_var, double* rewards, double* adv, int* valid,
                             cudaStream_t st) {
    if (n_groups <= 0) return;
    if (g < 2) throw std::invalid_argument("standardize_advantages: need G >= 2");
    const int n = n_groups * g;
    rewards_kernel<<<(n + 127) / 128, 128, 0, st>>>(n, tok, stride, len, plen, answer, g, rewards);
    SGB_KCHECK();
    advantages_kernel<<<(n_groups + 127) / 128, 128, 0, st>>>(n_groups, g, rewards, eps_var, adv, valid);
    SGB_KCHECK();
}

}  // namespace sgb
