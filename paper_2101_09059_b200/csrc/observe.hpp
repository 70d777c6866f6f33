// observe.hpp -- launchers of observe.cu (stress recovery, ensemble statistics).
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime_api.h>

namespace ens {

// out[F][6][n_s]: frame 0 (s_xx, s_yy, t_xy, t_xz, t_yz, 0) local shell; frame 1
// (s_rr, s_tt, s_zz, s_tz, s_rz, s_rt) in the basis M (rows b_p in local coordinates).
cudaError_t launch_stress(int64_t F, int32_t n_s, int32_t frame, const int32_t* etri, const double* G,
                          const double* M, const double* Ebar, double nu, double k_shear, const double* u,
                          double* out, cudaStream_t st);
// [rows][w][n_s] -> [n_s][rows][w] with row r written at map[r] (map may be null)
cudaError_t launch_to_abi(int64_t rows, int32_t w, int32_t n_s, const int32_t* map, const double* src, double* dst,
                          cudaStream_t st);
cudaError_t launch_magnitude(int64_t V, int32_t n_s, const double* u, double* mag, cudaStream_t st);
// mean / 5% / 95% over each length-n_s segment of values[n_seg][n_s]; segment k (row
// r = k / w, column k % w) is written at index map[r] * stride + offset + k % w.
size_t stats_temp_bytes(int64_t n_seg, int32_t n_s);
cudaError_t ensemble_stats(int64_t n_seg, int32_t n_s, int32_t w, const int32_t* map, int32_t stride,
                           int32_t offset, const double* values, double* sorted, void* temp, size_t temp_bytes,
                           double* mean, double* q05, double* q95, cudaStream_t st);

}  // namespace ens
