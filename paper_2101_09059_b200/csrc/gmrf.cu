// gmrf.cu -- GPU Matérn sampler: multi-right-hand-side Jacobi-PCG
// for A x = C~^{1/2} z, A = kappa^2 C~ + G (P1 lumped mass and stiffness on the wall mesh,
// Eqs. 4-6), so that x / sigma_SPDE has covariance Q_2^-1 exactly
// (Q_2 = A C~^-1 A, Eq. 4 with alpha = 2) — the same draw as the Cholesky route of
// Eq. 11 without a sparse factorisation.  All n_rhs systems advance
// together (realisation innermost), like the ensemble step itself; every reduction is a
// fixed-order two-stage sum, so results are run-to-run deterministic.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "gmrf.hpp"

namespace ens {
namespace {

constexpr int kT = 256;
constexpr int kRowsPerBlock = 64;     // rows reduced by one CTA for the per-column dots

// y = A x, A scalar CSR (RCM rows), x, y [V][n]
__global__ void k_spmm_scalar(int64_t V, int32_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ col,
                              const double* __restrict__ val, const double* __restrict__ x, double* __restrict__ y) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= V * n) return;
    const int64_t i = tid / n;
    const int s = int(tid - i * n);
    double acc = 0.0;
    for (int32_t k = rp[i]; k < rp[i + 1]; ++k) acc = fma(val[k], x[int64_t(col[k]) * n + s], acc);
    y[tid] = acc;
}

// partial[b][s] = sum over the block's rows of a[i][s] * c[i][s] (* d[i] if d)
__global__ void k_dot_partial(int64_t V, int32_t n, const double* __restrict__ a, const double* __restrict__ c,
                              const double* __restrict__ d, double* __restrict__ partial) {
    const int s = int(blockIdx.y) * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const int64_t i0 = int64_t(blockIdx.x) * kRowsPerBlock;
    const int64_t i1 = i0 + kRowsPerBlock < V ? i0 + kRowsPerBlock : V;
    double acc = 0.0;
    for (int64_t i = i0; i < i1; ++i) {
        const double t = a[i * n + s] * c[i * n + s];
        acc = d ? fma(t, d[i], acc) : acc + t;
    }
    partial[int64_t(blockIdx.x) * n + s] = acc;
}

__global__ void k_dot_final(int64_t nb, int32_t n, const double* __restrict__ partial, double* __restrict__ out) {
    const int s = int(blockIdx.x) * blockDim.x + threadIdx.x;
    if (s >= n) return;
    double acc = 0.0;
    for (int64_t b = 0; b < nb; ++b) acc += partial[b * n + s];
    out[s] = acc;
}

// x += alpha p; r -= alpha q  (alpha = rz / pq per column; frozen columns untouched)
__global__ void k_update_xr(int64_t V, int32_t n, const double* __restrict__ rz, const double* __restrict__ pq,
                            const int* __restrict__ active, const double* __restrict__ p, const double* __restrict__ q,
                            double* __restrict__ x, double* __restrict__ r) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= V * n) return;
    const int s = int(tid % n);
    if (!active[s]) return;
    const double al = rz[s] / pq[s];
    x[tid] = fma(al, p[tid], x[tid]);
    r[tid] = fma(-al, q[tid], r[tid]);
}

// z = D^-1 r
__global__ void k_precond(int64_t V, int32_t n, const double* __restrict__ dinv, const double* __restrict__ r,
                          double* __restrict__ z) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= V * n) return;
    z[tid] = dinv[tid / n] * r[tid];
}

// p = z + (rz_new / rz_old) p
__global__ void k_update_p(int64_t V, int32_t n, const double* __restrict__ rz_new, const double* __restrict__ rz_old,
                           const int* __restrict__ active, const double* __restrict__ z, double* __restrict__ p) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= V * n) return;
    const int s = int(tid % n);
    if (!active[s]) return;
    p[tid] = fma(rz_new[s] / rz_old[s], p[tid], z[tid]);
}

// b[i][s] = sqrt(C~_i) z[s][perm[i]] (ABI -> RCM rows); x_out[s][perm[i]] = scale x[i][s]
__global__ void k_rhs(int64_t V, int32_t n, const int32_t* __restrict__ perm, const double* __restrict__ sqrtC,
                      const double* __restrict__ z_abi, double* __restrict__ b) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= V * n) return;
    const int64_t i = tid / n;
    const int s = int(tid - i * n);
    b[tid] = sqrtC[i] * z_abi[int64_t(s) * V + perm[i]];
}

__global__ void k_out(int64_t V, int32_t n, const int32_t* __restrict__ perm, double scale, const double* __restrict__ x,
                      double* __restrict__ x_abi) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= V * n) return;
    const int64_t i = tid / n;
    const int s = int(tid - i * n);
    x_abi[int64_t(s) * V + perm[i]] = scale * x[tid];
}

inline unsigned gf(int64_t n) { return unsigned((n + kT - 1) / kT); }

}  // namespace

cudaError_t gmrf_pcg(const GmrfSystem& S, int32_t n, const double* d_z_abi, double* d_x_abi, double scale, double tol,
                     int32_t max_iter, double* work, cudaStream_t st, int32_t* iters, double* max_rel_res) {
    const int64_t V = S.V, Vn = V * n;
    double* x = work;
    double* r = x + Vn;
    double* z = r + Vn;
    double* p = z + Vn;
    double* q = p + Vn;
    const int64_t nb = (V + kRowsPerBlock - 1) / kRowsPerBlock;
    double* partial = q + Vn;                    // [nb][n]
    double* rz = partial + nb * n;               // [n] each
    double* rz_new = rz + n;
    double* pq = rz_new + n;
    double* bb = pq + n;
    double* rr = bb + n;
    int* d_active = reinterpret_cast<int*>(rr + n);
    const dim3 dgrid(unsigned(nb), unsigned((n + kT - 1) / kT));
    auto dot = [&](const double* a, const double* c, const double* d, double* out) {
        k_dot_partial<<<dgrid, kT, 0, st>>>(V, n, a, c, d, partial);
        k_dot_final<<<gf(n), kT, 0, st>>>(nb, n, partial, out);
        return cudaGetLastError();
    };
    cudaError_t e;
    k_rhs<<<gf(Vn), kT, 0, st>>>(V, n, S.perm, S.sqrtC, d_z_abi, r);      // r = b (x0 = 0)
    if ((e = cudaMemsetAsync(x, 0, size_t(Vn) * sizeof(double), st))) return e;
    if ((e = dot(r, r, nullptr, bb))) return e;
    k_precond<<<gf(Vn), kT, 0, st>>>(V, n, S.dinv, r, z);
    if ((e = cudaMemcpyAsync(p, z, size_t(Vn) * sizeof(double), cudaMemcpyDeviceToDevice, st))) return e;
    if ((e = dot(r, z, nullptr, rz))) return e;
    std::vector<double> h_bb(static_cast<size_t>(n)), h_rr(static_cast<size_t>(n));
    std::vector<int> active(size_t(n), 1);
    if ((e = cudaMemcpyAsync(h_bb.data(), bb, size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, st))) return e;
    if ((e = cudaStreamSynchronize(st))) return e;
    for (int s = 0; s < n; ++s)
        if (!(h_bb[size_t(s)] > 0.0)) active[size_t(s)] = 0;
    if ((e = cudaMemcpyAsync(d_active, active.data(), size_t(n) * sizeof(int), cudaMemcpyHostToDevice, st))) return e;
    int it = 0;
    double worst = 0.0;
    for (; it < max_iter; ++it) {
        k_spmm_scalar<<<gf(Vn), kT, 0, st>>>(V, n, S.rp, S.col, S.val, p, q);
        if ((e = dot(p, q, nullptr, pq))) return e;
        k_update_xr<<<gf(Vn), kT, 0, st>>>(V, n, rz, pq, d_active, p, q, x, r);
        k_precond<<<gf(Vn), kT, 0, st>>>(V, n, S.dinv, r, z);
        if ((e = dot(r, z, nullptr, rz_new))) return e;
        k_update_p<<<gf(Vn), kT, 0, st>>>(V, n, rz_new, rz, d_active, z, p);
        if ((e = cudaMemcpyAsync(rz, rz_new, size_t(n) * sizeof(double), cudaMemcpyDeviceToDevice, st))) return e;
        if (it % 10 == 9 || it + 1 == max_iter) {                         // convergence check
            if ((e = dot(r, r, nullptr, rr))) return e;
            if ((e = cudaMemcpyAsync(h_rr.data(), rr, size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, st))) return e;
            if ((e = cudaStreamSynchronize(st))) return e;
            bool any = false;
            worst = 0.0;
            for (int s = 0; s < n; ++s) {
                const double rel = h_bb[size_t(s)] > 0 ? std::sqrt(h_rr[size_t(s)] / h_bb[size_t(s)]) : 0.0;
                worst = std::max(worst, rel);
                if (active[size_t(s)] && rel <= tol) active[size_t(s)] = 0;
                any = any || active[size_t(s)];
            }
            if (!any) {
                ++it;
                break;
            }
            if ((e = cudaMemcpyAsync(d_active, active.data(), size_t(n) * sizeof(int), cudaMemcpyHostToDevice, st)))
                return e;
        }
    }
    k_out<<<gf(Vn), kT, 0, st>>>(V, n, S.perm, scale, x, d_x_abi);
    if ((e = cudaGetLastError())) return e;
    if ((e = cudaStreamSynchronize(st))) return e;
    if (iters) *iters = it;
    if (max_rel_res) *max_rel_res = worst;
    return cudaSuccess;
}

size_t gmrf_work_doubles(int64_t V, int32_t n) {
    const int64_t nb = (V + kRowsPerBlock - 1) / kRowsPerBlock;
    return size_t(5 * V * n + nb * n + 5 * n) + size_t(n);     // + int flags (<= n doubles)
}

}  // namespace ens
