// Host-side error plumbing shared by the C-ABI and the engine.
#pragma once

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <stdexcept>
#include <string>

namespace sgb {

// Status codes of the C-ABI (include/sgrpo_b200.h). They map 1:1 onto the exception
// types of the reference's C++ API (SURVEY.md §8b error conventions).
enum Status : int {
    SGB_OK = 0,
    SGB_EINVAL = 1,    // std::invalid_argument
    SGB_ERANGE = 2,    // std::out_of_range
    SGB_ERUNTIME = 3,  // std::runtime_error
    SGB_EDOMAIN = 4,   // std::domain_error
    SGB_ECUDA = 5,     // CUDA failure (no CPU fallback exists)
};

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

// NVTX ranges around the engine's phases (rollout, prefill, step, draft, verify, accept,
// draft / policy update): visible in Nsight Systems / Compute timelines, a no-op without a tool
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

#define SGB_CUDA(x) ::sgb::cuda_check((x), #x)
#define SGB_KCHECK() ::sgb::cuda_check(cudaGetLastError(), "kernel launch")

}  // namespace sgb
