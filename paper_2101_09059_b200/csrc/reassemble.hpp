// reassemble.hpp -- launcher of reassemble.cu (geometry-updated stiffness, N4).
#pragma once

#include <cstdint>
#include <cuda_runtime_api.h>

namespace ens {

// Kval[b][9][n_s] of the nblk stored blocks from the element contributions (cptr/contrib as
// F0: code = local element * 9 + a * 3 + b'), alpha [F_loc][n_s], local element node ids
// etri [F_loc][3], local node coordinates xyz [n_loc][3] and displacement u [n_loc][3][n_s].
cudaError_t launch_reassemble(int64_t nblk, int32_t n_s, const int32_t* cptr, const int32_t* contrib,
                              const double* alpha, const int32_t* etri, const double* xyz, const double* u, double nu,
                              double k_shear, double* Kval, cudaStream_t st);

}  // namespace ens
