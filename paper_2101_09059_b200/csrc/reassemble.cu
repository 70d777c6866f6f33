// reassemble.cu -- selective stiffness re-assembly on the updated geometry (SURVEY.md §8(f)
// N4).  Every k steps each realisation's stored block values are rebuilt from
// its own deformed nodes X + u_n^s: Kval[b][c][d][s] = sum over the block's element
// contributions (ascending element, as F0) of alpha[e][s] K^_e(X + u^s)[3a+c][3b'+d], with
// the K^ sub-block in the closed form of host_setup.cpp element_stiffness.  Entries below
// the 9x9 diagonal are taken from the mirrored upper entry, so the rebuilt K_s stays
// exactly symmetric (the half-storage kernel relies on it).
#include <cstdint>

#include <cuda_runtime.h>

#include "reassemble.hpp"

namespace ens {
namespace {

constexpr int kT = 256;

// Upper-triangle entry (r <= q of the element's 9x9) of K^ for E = 1, unit thickness.
struct ElemFrame {
    double e[3][3];   // rows e1, e2, e3
    double b[3], c[3];
    double q, g, nu, ks;
};

__device__ __forceinline__ void elem_frame(const double (&X)[3][3], double nu, double ks, ElemFrame& F) {
    const double d21[3] = {X[1][0] - X[0][0], X[1][1] - X[0][1], X[1][2] - X[0][2]};
    const double d31[3] = {X[2][0] - X[0][0], X[2][1] - X[0][1], X[2][2] - X[0][2]};
    const double n[3] = {d21[1] * d31[2] - d21[2] * d31[1], d21[2] * d31[0] - d21[0] * d31[2],
                         d21[0] * d31[1] - d21[1] * d31[0]};
    const double nn = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    const double l = sqrt(d21[0] * d21[0] + d21[1] * d21[1] + d21[2] * d21[2]);
    const double A = 0.5 * nn;
    for (int k = 0; k < 3; ++k) {
        F.e[0][k] = d21[k] / l;
        F.e[2][k] = n[k] / nn;
    }
    F.e[1][0] = F.e[2][1] * F.e[0][2] - F.e[2][2] * F.e[0][1];
    F.e[1][1] = F.e[2][2] * F.e[0][0] - F.e[2][0] * F.e[0][2];
    F.e[1][2] = F.e[2][0] * F.e[0][1] - F.e[2][1] * F.e[0][0];
    double x[3], y[3];
    for (int a = 0; a < 3; ++a) {
        const double d[3] = {X[a][0] - X[0][0], X[a][1] - X[0][1], X[a][2] - X[0][2]};
        x[a] = d[0] * F.e[0][0] + d[1] * F.e[0][1] + d[2] * F.e[0][2];
        y[a] = d[0] * F.e[1][0] + d[1] * F.e[1][1] + d[2] * F.e[1][2];
    }
    F.b[0] = y[1] - y[2]; F.b[1] = y[2] - y[0]; F.b[2] = y[0] - y[1];
    F.c[0] = x[2] - x[1]; F.c[1] = x[0] - x[2]; F.c[2] = x[1] - x[0];
    const double pre = 1.0 / (1.0 - nu * nu);
    F.g = 0.5 * (1.0 - nu);
    F.q = pre / (4.0 * A);
    F.nu = nu;
    F.ks = ks;
}

// global entry (r, col) of K^, r <= col (r = 3a+i, col = 3bb+j)
__device__ __forceinline__ double khat_upper(const ElemFrame& F, int r, int col) {
    const int a = r / 3, i = r % 3, bb = col / 3, j = col % 3;
    const double q = F.q, g = F.g, nu = F.nu;
    const double kl[3][3] = {
        {q * (F.b[a] * F.b[bb] + g * F.c[a] * F.c[bb]), q * (nu * F.b[a] * F.c[bb] + g * F.c[a] * F.b[bb]), 0.0},
        {q * (nu * F.c[a] * F.b[bb] + g * F.b[a] * F.c[bb]), q * (F.c[a] * F.c[bb] + g * F.b[a] * F.b[bb]), 0.0},
        {0.0, 0.0, q * g * F.ks * (F.b[a] * F.b[bb] + F.c[a] * F.c[bb])}};
    double s = 0.0;
    for (int p = 0; p < 3; ++p)
        for (int t = 0; t < 3; ++t) s += F.e[p][i] * kl[p][t] * F.e[t][j];
    return s;
}

__global__ void __launch_bounds__(kT)
k_reassemble(int64_t nblk, int32_t n_s, const int32_t* __restrict__ cptr, const int32_t* __restrict__ contrib,
             const double* __restrict__ alpha, const int32_t* __restrict__ etri, const double* __restrict__ xyz,
             const double* __restrict__ u, double nu, double ks, double* __restrict__ Kval) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= nblk * n_s) return;
    const int64_t blk = tid / n_s;
    const int s = int(tid - blk * n_s);
    double acc[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) acc[k] = 0.0;
    for (int32_t q = cptr[blk]; q < cptr[blk + 1]; ++q) {
        const int32_t code = contrib[q];
        const int64_t e = code / 9;
        const int ab = code % 9, la = ab / 3, lb = ab % 3;
        double X[3][3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const int64_t node = etri[3 * e + a];
#pragma unroll
            for (int d = 0; d < 3; ++d) X[a][d] = xyz[3 * node + d] + u[(node * 3 + d) * n_s + s];
        }
        ElemFrame F;
        elem_frame(X, nu, ks, F);
        const double al = alpha[e * n_s + s];
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const int r = 3 * la + c, col = 3 * lb + d;
                const double kv = r <= col ? khat_upper(F, r, col) : khat_upper(F, col, r);
                acc[3 * c + d] = fma(al, kv, acc[3 * c + d]);
            }
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) Kval[(blk * 9 + k) * n_s + s] = acc[k];
}

}  // namespace

cudaError_t launch_reassemble(int64_t nblk, int32_t n_s, const int32_t* cptr, const int32_t* contrib,
                              const double* alpha, const int32_t* etri, const double* xyz, const double* u, double nu,
                              double k_shear, double* Kval, cudaStream_t st) {
    const int64_t n = nblk * n_s;
    if (n == 0) return cudaSuccess;
    k_reassemble<<<unsigned((n + kT - 1) / kT), kT, 0, st>>>(nblk, n_s, cptr, contrib, alpha, etri, xyz, u, nu, k_shear,
                                                              Kval);
    return cudaGetLastError();
}

}  // namespace ens
