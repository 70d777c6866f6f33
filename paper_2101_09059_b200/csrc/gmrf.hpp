// gmrf.hpp -- multi-RHS Jacobi-PCG for the SPDE/GMRF sampler (gmrf.cu).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime_api.h>

namespace ens {

struct GmrfSystem {
    int64_t V = 0;
    const int32_t* rp = nullptr;      // scalar CSR of A = kappa^2 C~ + G in RCM order
    const int32_t* col = nullptr;
    const double* val = nullptr;
    const double* dinv = nullptr;     // 1 / diag(A)
    const double* sqrtC = nullptr;    // sqrt(C~_i)
    const int32_t* perm = nullptr;    // RCM row -> caller node
};

// x_abi[s][node] = scale * (A^-1 sqrt(C~) z_abi[s])[node] for s < n; work has
// gmrf_work_doubles(V, n) doubles.  Stops when every column's relative residual <= tol.
cudaError_t gmrf_pcg(const GmrfSystem& S, int32_t n, const double* d_z_abi, double* d_x_abi, double scale, double tol,
                     int32_t max_iter, double* work, cudaStream_t st, int32_t* iters, double* max_rel_res);
size_t gmrf_work_doubles(int64_t V, int32_t n);

}  // namespace ens
