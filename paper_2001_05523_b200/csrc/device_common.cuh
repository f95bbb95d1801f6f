// Device-side helpers shared by the quadrature and matvec kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "h2b_internal.h"

#define H2B_CUDA_TRY(expr)                                                                     \
    do {                                                                                       \
        cudaError_t _e = (expr);                                                               \
        if (_e != cudaSuccess)                                                                 \
            return h2b::fail(H2B_ERR_CUDA, std::string(#expr " failed: ") + cudaGetErrorString(_e)); \
    } while (0)

namespace h2b {

constexpr double kPi = 3.141592653589793238462643383279502884;
constexpr double kInv4Pi = 1.0 / (4.0 * kPi);

// Hardware reciprocal-square-root seed (MUFU.RSQ64H); refined by one Newton
// step at every call site, folded into the quadrature accumulation.
__device__ __forceinline__ double rsqrt_seed(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace h2b
