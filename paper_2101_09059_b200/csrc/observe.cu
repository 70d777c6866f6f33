// observe.cu -- S6 observation and the next row of the scope table:
// element stresses in the local shell frame or the paper's centreline frame
// and ensemble statistics (mean, 5%/95% quantiles over the
// realisations) computed on the device from the resident state.
// Off the hot path; CUB's segmented sort is used as a library primitive.
#include <algorithm>
#include <cstdint>

#include <cub/device/device_segmented_sort.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>
#include <cuda_runtime.h>

#include "observe.hpp"

namespace ens {
namespace {

constexpr int kT = 256;
inline unsigned grid_for(int64_t n) { return unsigned((n + kT - 1) / kT); }

// thread = (element e, realisation s); out [F][6][n_s]
__global__ void k_stress(int64_t F, int32_t n_s, int32_t frame, const int32_t* __restrict__ etri,
                         const double* __restrict__ G, const double* __restrict__ M,
                         const double* __restrict__ Ebar, double nu, double ks, const double* __restrict__ u,
                         double* __restrict__ out) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= F * n_s) return;
    const int64_t e = tid / n_s;
    const int s = int(tid - e * n_s);
    double ue[9];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int64_t node = etri[3 * e + a];
#pragma unroll
        for (int d = 0; d < 3; ++d) ue[3 * a + d] = u[(node * 3 + d) * n_s + s];
    }
    const double* g = G + e * 45;
    double eps[5];
#pragma unroll
    for (int r = 0; r < 5; ++r) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < 9; ++k) acc = fma(g[9 * r + k], ue[k], acc);
        eps[r] = acc;
    }
    const double pre = Ebar[e * n_s + s] / (1.0 - nu * nu);
    const double sxx = pre * (eps[0] + nu * eps[1]);
    const double syy = pre * (nu * eps[0] + eps[1]);
    const double txy = pre * 0.5 * (1.0 - nu) * eps[2];
    const double txz = pre * 0.5 * ks * (1.0 - nu) * eps[3];
    const double tyz = pre * 0.5 * ks * (1.0 - nu) * eps[4];
    double o[6];
    if (frame == 0) {
        o[0] = sxx; o[1] = syy; o[2] = txy; o[3] = txz; o[4] = tyz; o[5] = 0.0;
    } else {
        const double S[3][3] = {{sxx, txy, txz}, {txy, syy, tyz}, {txz, tyz, 0.0}};
        const double* m = M + e * 9;
        double Sc[3][3];
#pragma unroll
        for (int p = 0; p < 3; ++p)
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                double acc = 0.0;
#pragma unroll
                for (int i = 0; i < 3; ++i)
#pragma unroll
                    for (int j = 0; j < 3; ++j) acc = fma(m[3 * p + i] * S[i][j], m[3 * q + j], acc);
                Sc[p][q] = acc;
            }
        o[0] = Sc[0][0]; o[1] = Sc[1][1]; o[2] = Sc[2][2]; o[3] = Sc[1][2]; o[4] = Sc[0][2]; o[5] = Sc[0][1];
    }
#pragma unroll
    for (int c = 0; c < 6; ++c) out[(e * 6 + c) * n_s + s] = o[c];
}

// [rows][w][n_s] (device) -> [n_s][rows][w] (ABI), rows in map order
__global__ void k_to_abi(int64_t rows, int32_t w, int32_t n_s, const int32_t* __restrict__ map,
                         const double* __restrict__ src, double* __restrict__ dst) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= rows * w * n_s) return;
    const int s = int(tid % n_s);
    const int64_t rc = tid / n_s;
    const int64_t r = rc / w;
    const int c = int(rc - r * w);
    const int64_t ro = map ? map[r] : r;
    dst[(int64_t(s) * rows + ro) * w + c] = src[tid];
}

// |u| per (node, realisation): [V][n_s]
__global__ void k_magnitude(int64_t V, int32_t n_s, const double* __restrict__ u, double* __restrict__ mag) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= V * n_s) return;
    const int64_t i = tid / n_s;
    const int s = int(tid - i * n_s);
    const double x = u[(i * 3) * n_s + s], y = u[(i * 3 + 1) * n_s + s], z = u[(i * 3 + 2) * n_s + s];
    mag[tid] = sqrt(fma(x, x, fma(y, y, z * z)));
}

// from sorted segments: mean (ascending summation) and quantiles p by linear interpolation
// between order statistics, h = (n - 1) p.  out row = map[seg / w] * w + seg % w.
__global__ void k_quantiles(int64_t n_seg, int32_t n_s, int32_t w, const int32_t* __restrict__ map,
                            int32_t stride, int32_t offset, const double* __restrict__ sorted,
                            double* __restrict__ mean, double* __restrict__ q05, double* __restrict__ q95) {
    const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= n_seg) return;
    const double* v = sorted + k * n_s;
    double acc = 0.0;
    for (int i = 0; i < n_s; ++i) acc += v[i];
    const int64_t r = k / w;
    const int64_t o = (map ? map[r] : r) * stride + offset + (k - r * w);
    mean[o] = acc / n_s;
    const double ps[2] = {0.05, 0.95};
    double* outs[2] = {q05, q95};
    for (int j = 0; j < 2; ++j) {
        const double h = (n_s - 1) * ps[j];
        const int lo = int(floor(h));
        const int hi = lo + 1 < n_s ? lo + 1 : n_s - 1;
        outs[j][o] = v[lo] + (h - lo) * (v[hi] - v[lo]);
    }
}

struct SegOffset {
    int32_t n_s;
    __host__ __device__ int operator()(int k) const { return k * n_s; }
};

}  // namespace

cudaError_t launch_stress(int64_t F, int32_t n_s, int32_t frame, const int32_t* etri, const double* G,
                          const double* M, const double* Ebar, double nu, double k_shear, const double* u,
                          double* out, cudaStream_t st) {
    if (F * n_s == 0) return cudaSuccess;
    k_stress<<<grid_for(F * n_s), kT, 0, st>>>(F, n_s, frame, etri, G, M, Ebar, nu, k_shear, u, out);
    return cudaGetLastError();
}

cudaError_t launch_to_abi(int64_t rows, int32_t w, int32_t n_s, const int32_t* map, const double* src, double* dst,
                          cudaStream_t st) {
    if (rows * w * n_s == 0) return cudaSuccess;
    k_to_abi<<<grid_for(rows * w * n_s), kT, 0, st>>>(rows, w, n_s, map, src, dst);
    return cudaGetLastError();
}

cudaError_t launch_magnitude(int64_t V, int32_t n_s, const double* u, double* mag, cudaStream_t st) {
    if (V * n_s == 0) return cudaSuccess;
    k_magnitude<<<grid_for(V * n_s), kT, 0, st>>>(V, n_s, u, mag);
    return cudaGetLastError();
}

size_t stats_temp_bytes(int64_t n_seg, int32_t n_s) {
    const int64_t per = std::max<int64_t>(1, (int64_t(1) << 30) / n_s);     // segments per CUB call
    const int seg = int(std::min<int64_t>(n_seg, per));
    size_t bytes = 0;
    auto off = thrust::make_transform_iterator(thrust::counting_iterator<int>(0), SegOffset{n_s});
    cub::DeviceSegmentedSort::SortKeys(nullptr, bytes, static_cast<const double*>(nullptr), static_cast<double*>(nullptr),
                                       seg * n_s, seg, off, off + 1);
    return bytes + 256;
}

cudaError_t ensemble_stats(int64_t n_seg, int32_t n_s, int32_t w, const int32_t* map, int32_t stride,
                           int32_t offset, const double* values, double* sorted, void* temp, size_t temp_bytes,
                           double* mean, double* q05, double* q95, cudaStream_t st) {
    const int64_t per = std::max<int64_t>(1, (int64_t(1) << 30) / n_s);
    for (int64_t k0 = 0; k0 < n_seg; k0 += per) {
        const int seg = int(std::min<int64_t>(per, n_seg - k0));
        auto off = thrust::make_transform_iterator(thrust::counting_iterator<int>(0), SegOffset{n_s});
        size_t bytes = temp_bytes;
        cudaError_t e = cub::DeviceSegmentedSort::SortKeys(temp, bytes, values + k0 * n_s, sorted + k0 * n_s,
                                                           seg * n_s, seg, off, off + 1, st);
        if (e != cudaSuccess) return e;
    }
    k_quantiles<<<grid_for(n_seg), kT, 0, st>>>(n_seg, n_s, w, map, stride, offset, sorted, mean, q05, q95);
    return cudaGetLastError();
}

}  // namespace ens
