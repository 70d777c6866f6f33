// kernels.cu -- sm_100a kernels of the ensemble explicit shell step (arXiv 2101.09059).
//
// Hot path (north star): r = f_ext - K(theta_s) u_s over N_s realisations, fused with the
// central-difference update (Eq. 22).  fp64 throughout, CUDA cores:
// this is a sparse streaming product, not a dense contraction, so no tensor cores.
//
// Thread mapping (assembled kernel): thread = (row i, realisation group g), VEC
// consecutive realisations per thread, groups of one row on consecutive lanes, so that
// every (block, entry) segment Kval[b][k][0..n_s) — n_s*8 contiguous bytes — is read by
// consecutive lanes with 16 B (VEC = 2) or 32 B (VEC = 4) vector loads.  Each thread
// accumulates its realisations sequentially in CSR block order then d = 0,1,2 with explicit
// fma(): the per-realisation arithmetic is identical whatever N_s, VEC or the launch
// geometry, which makes ensemble runs bit-identical to single-realisation runs.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "device.hpp"

namespace ens {
namespace {

constexpr int kThreads = 256;

struct d4 { double x, y, z, w; };

template <int VEC> struct Vec;
template <> struct Vec<1> { double v[1]; };
template <> struct Vec<2> { double v[2]; };
template <> struct Vec<4> { double v[4]; };

// ---- loads -----------------------------------------------------------------------------
// Kval is streamed exactly once per step: no L1 allocation, L2 evict-first (createpolicy /
// the 256-bit EFL2 form), so the u_n gather working set stays resident in the 126 MB L2.
template <int VEC>
__device__ __forceinline__ Vec<VEC> ld_stream(const double* p, uint64_t pol);

template <>
__device__ __forceinline__ Vec<1> ld_stream<1>(const double* p, uint64_t pol) {
    Vec<1> r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
                 : "=d"(r.v[0]) : "l"(p), "l"(pol));
    return r;
}
template <>
__device__ __forceinline__ Vec<2> ld_stream<2>(const double* p, uint64_t pol) {
    Vec<2> r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(r.v[0]), "=d"(r.v[1]) : "l"(p), "l"(pol));
    return r;
}
template <>
__device__ __forceinline__ Vec<4> ld_stream<4>(const double* p, uint64_t) {
    Vec<4> r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::evict_first.v4.f64 {%0, %1, %2, %3}, [%4];"
                 : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3]) : "l"(p));
    return r;
}

// Symmetric storage: each stored block is read twice (by its row and, transposed, by its
// column's row within the RCM bandwidth), so no L1 allocation but the normal L2 policy.
template <int VEC>
__device__ __forceinline__ Vec<VEC> ld_once_l1(const double* p) {
    Vec<VEC> r;
    if constexpr (VEC == 1) {
        asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r.v[0]) : "l"(p));
    } else if constexpr (VEC == 2) {
        asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.v[0]), "=d"(r.v[1]) : "l"(p));
    } else {
        asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
                     : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3]) : "l"(p));
    }
    return r;
}

// u_n and the coefficient arrays: read-only within a launch, re-used across rows via L1/L2.
template <int VEC>
__device__ __forceinline__ Vec<VEC> ld_ro(const double* p) {
    Vec<VEC> r;
    if constexpr (VEC == 1) {
        r.v[0] = __ldg(p);
    } else if constexpr (VEC == 2) {
        double2 t = __ldg(reinterpret_cast<const double2*>(p));
        r.v[0] = t.x; r.v[1] = t.y;
    } else {
        asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"
                     : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3]) : "l"(p));
    }
    return r;
}

// u_{n-1}: read then overwritten in place by the same thread (plain coherent accesses).
template <int VEC>
__device__ __forceinline__ Vec<VEC> ld_rw(const double* p) {
    Vec<VEC> r;
    if constexpr (VEC == 1) {
        r.v[0] = *p;
    } else if constexpr (VEC == 2) {
        double2 t = *reinterpret_cast<const double2*>(p);
        r.v[0] = t.x; r.v[1] = t.y;
    } else {
        asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
                     : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3]) : "l"(p));
    }
    return r;
}

template <int VEC>
__device__ __forceinline__ void st_vec(double* p, const Vec<VEC>& x) {
    if constexpr (VEC == 1) {
        *p = x.v[0];
    } else if constexpr (VEC == 2) {
        *reinterpret_cast<double2*>(p) = make_double2(x.v[0], x.v[1]);
    } else {
        asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};"
                     :: "l"(p), "d"(x.v[0]), "d"(x.v[1]), "d"(x.v[2]), "d"(x.v[3]) : "memory");
    }
}

// ---- load coefficients coef_k = ramp(t) g_k(t)  (ens_set_traction contract) ------------
__device__ void load_coeffs(const StepArgs& a, double t, double* coef) {
    double ramp = 1.0;
    if (a.ramp_T > 0.0 && t < a.ramp_T) ramp = sin(3.141592653589793 * t / (2.0 * a.ramp_T));
    double tau = t;
    if (a.period > 0.0) tau = t - a.period * floor(t / a.period);
    for (int k = 0; k < a.n_fields; ++k) {
        double g = 1.0;
        if (a.n_tab > 0) {
            const double* G = a.tab_g + int64_t(k) * a.n_tab;
            if (tau <= a.tab_t[0]) {
                g = G[0];
            } else if (tau >= a.tab_t[a.n_tab - 1]) {
                g = G[a.n_tab - 1];
            } else {
                int lo = 0, hi = a.n_tab - 1;          // tab_t[lo] <= tau < tab_t[hi]
                while (hi - lo > 1) {
                    int mid = (lo + hi) >> 1;
                    if (a.tab_t[mid] <= tau) lo = mid; else hi = mid;
                }
                g = G[lo] + (G[lo + 1] - G[lo]) * (tau - a.tab_t[lo]) / (a.tab_t[lo + 1] - a.tab_t[lo]);
            }
        }
        coef[k] = ramp * g;
    }
}

struct StepCtx {
    int64_t step;
    const double* un;
    double* uo;       // u_{n-1} in, u_{n+1} out
};

__device__ __forceinline__ StepCtx step_ctx(const StepArgs& a) {
    StepCtx c;
    c.step = *a.step_base + a.step_off;
    c.un = (c.step & 1) ? a.ubuf1 : a.ubuf0;
    c.uo = (c.step & 1) ? a.ubuf0 : a.ubuf1;
    return c;
}

// S2 + S4: r = f - y; u_{n+1} = c1 r + c2 u_n - c3 u_{n-1}; Dirichlet; non-finite flag.
// The operands of the update do not depend on the product, so they are loaded (upd_load)
// before the gather loop and their latency hides behind it; upd_store finishes the step.
template <int VEC>
struct Upd {
    Vec<VEC> c1, c2, c3, un[3], uo[3];
    double f[3];
    uint8_t fx;
};

template <int VEC>
__device__ __forceinline__ void upd_load(const StepArgs& a, const StepCtx& sc, const double* coef, int64_t i,
                                         int s0, Upd<VEC>& u, bool load_un) {
    const int n_s = a.n_s;
    u.fx = a.fixed ? __ldg(a.fixed + i) : uint8_t(0);
    u.c1 = ld_ro<VEC>(a.c1 + i * n_s + s0);
    if (a.c2a) {
        u.c2 = ld_ro<VEC>(a.c2a + i * n_s + s0);
        u.c3 = ld_ro<VEC>(a.c3a + i * n_s + s0);
    } else {
#pragma unroll
        for (int v = 0; v < VEC; ++v) { u.c2.v[v] = a.c2; u.c3.v[v] = a.c3; }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const int64_t off = (i * 3 + c) * n_s + s0;
        if (load_un) u.un[c] = ld_ro<VEC>(sc.un + off);
        u.uo[c] = ld_rw<VEC>(sc.uo + off);
        double f = 0.0;
        for (int k = 0; k < a.n_fields; ++k) f = fma(coef[k], __ldg(a.Fk + (int64_t(k) * a.fk_rows + i) * 3 + c), f);
        u.f[c] = f;
    }
}

// Register-free variant for the matrix-free kernel: cp.async (LDGSTS) copies c1 (c2, c3)
// and u_{n-1} of the thread's row into its shared-memory slot; read back after the gather.
template <int VEC>
__device__ __forceinline__ void cp_async_vec(double* dst_smem, const double* src) {
    const uint32_t d = uint32_t(__cvta_generic_to_shared(dst_smem));
    if constexpr (VEC == 1) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(d), "l"(src) : "memory");
    } else if constexpr (VEC == 2) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(d), "l"(src) : "memory");
    } else {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(d), "l"(src) : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(d + 16), "l"(src + 2) : "memory");
    }
}

template <int VEC>
__device__ __forceinline__ void upd_load_async(const StepArgs& a, const StepCtx& sc, int64_t i, int s0,
                                               double* slot /* 6 * VEC doubles */) {
    const int n_s = a.n_s;
    cp_async_vec<VEC>(slot, a.c1 + i * n_s + s0);
    if (a.c2a) {
        cp_async_vec<VEC>(slot + VEC, a.c2a + i * n_s + s0);
        cp_async_vec<VEC>(slot + 2 * VEC, a.c3a + i * n_s + s0);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) cp_async_vec<VEC>(slot + (3 + c) * VEC, sc.uo + (i * 3 + c) * n_s + s0);
    asm volatile("cp.async.commit_group;" ::: "memory");
}

template <int VEC>
__device__ __forceinline__ void upd_collect(const StepArgs& a, const double* coef, int64_t i, const double* slot,
                                            Upd<VEC>& u) {
    asm volatile("cp.async.wait_all;" ::: "memory");
    u.fx = a.fixed ? __ldg(a.fixed + i) : uint8_t(0);
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
        u.c1.v[v] = slot[v];
        u.c2.v[v] = a.c2a ? slot[VEC + v] : a.c2;
        u.c3.v[v] = a.c2a ? slot[2 * VEC + v] : a.c3;
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int v = 0; v < VEC; ++v) u.uo[c].v[v] = slot[(3 + c) * VEC + v];
        double f = 0.0;
        for (int k = 0; k < a.n_fields; ++k) f = fma(coef[k], __ldg(a.Fk + (int64_t(k) * a.fk_rows + i) * 3 + c), f);
        u.f[c] = f;
    }
}

template <int VEC>
__device__ __forceinline__ void upd_store(const StepArgs& a, const StepCtx& sc, int64_t i, int s0,
                                          const double (&y)[3][VEC], const Upd<VEC>& u) {
    const int n_s = a.n_s;
    unsigned bad = 0;   // bit v: realisation s0 + v produced a non-finite value
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        Vec<VEC> out;
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
            const double r = u.f[c] - y[c][v];
            const double t = fma(u.c2.v[v], u.un[c].v[v], -(u.c3.v[v] * u.uo[c].v[v]));
            double w = fma(u.c1.v[v], r, t);
            if ((u.fx >> c) & 1) w = 0.0;
            bad |= unsigned(!isfinite(w)) << v;
            out.v[v] = w;
        }
        st_vec<VEC>(sc.uo + (i * 3 + c) * n_s + s0, out);
    }
    if (bad) {
        for (int v = 0; v < VEC; ++v)
            if ((bad >> v) & 1) {
                unsigned long long code = (unsigned long long)(sc.step) << 24 | (unsigned long long)(a.s_global0 + s0 + v);
                atomicMin(a.flag, code);
            }
    }
}

template <int VEC>
__device__ __forceinline__ void store_y(const StepArgs& a, int64_t i, int s0, const double (&y)[3][VEC]) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        Vec<VEC> o;
#pragma unroll
        for (int v = 0; v < VEC; ++v) o.v[v] = y[c][v];
        st_vec<VEC>(a.y_out + (i * 3 + c) * a.n_s + s0, o);
    }
}

// ---- F1: fused step on the assembled per-realisation block values ----------------------
template <int VEC, bool APPLY, bool PREF>
__global__ void __launch_bounds__(kThreads)
k_step_assembled(const StepArgs a) {
    __shared__ double s_coef[kMaxFields];
    const StepCtx sc = step_ctx(a);
    if (!APPLY && threadIdx.x == 0) load_coeffs(a, double(sc.step) * a.dt, s_coef);
    if (!APPLY) __syncthreads();

    const int P = a.n_s / VEC;                       // realisation groups per row
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= a.V * P) return;
    const int64_t i = a.row0 + tid / P;
    const int s0 = int(tid % P) * VEC;
    const int n_s = a.n_s;

    uint64_t pol = 0;
    if constexpr (VEC < 4) asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));

    Upd<VEC> upd;
    if constexpr (!APPLY && PREF) upd_load<VEC>(a, sc, s_coef, i, s0, upd, true);

    double y[3][VEC];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int v = 0; v < VEC; ++v) y[c][v] = 0.0;

    const int32_t b_end = __ldg(a.row_ptr + i + 1);
#pragma unroll 2
    for (int32_t b = __ldg(a.row_ptr + i); b < b_end; ++b) {
        const int64_t j = __ldg(a.col + b);
        const double* kp = a.Kval + int64_t(b) * 9 * n_s + s0;
        const double* up = sc.un + j * 3 * n_s + s0;
        Vec<VEC> u[3], k[9];
#pragma unroll
        for (int d = 0; d < 3; ++d) u[d] = ld_ro<VEC>(up + d * n_s);
#pragma unroll
        for (int e = 0; e < 9; ++e) k[e] = ld_stream<VEC>(kp + e * n_s, pol);
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int d = 0; d < 3; ++d)
#pragma unroll
                for (int v = 0; v < VEC; ++v) y[c][v] = fma(k[3 * c + d].v[v], u[d].v[v], y[c][v]);
    }
    if constexpr (APPLY) {
        store_y<VEC>(a, i, s0, y);
    } else {
        if constexpr (!PREF) upd_load<VEC>(a, sc, s_coef, i, s0, upd, true);
        upd_store<VEC>(a, sc, i, s0, y, upd);
    }
}

// ---- F1s: fused step on symmetric (half) block storage ----------------------------------
// K_s is symmetric (Eq. 10: B^T C B), so only the blocks (i, j >= i) are stored; row i takes
// its blocks (i, j < i) as the transposes of blocks stored with row j (within the RCM
// bandwidth, so still in L2).  Lower references (j ascending) then the row's own upper
// blocks (j ascending) visit the columns in exactly the order of the full CSR row, and
// K^_e is exactly symmetric, so the result is bit-identical to F1 with ~half the bytes.
template <int VEC, bool APPLY, bool PREF>
__global__ void __launch_bounds__(kThreads)
k_step_assembled_sym(const StepArgs a) {
    __shared__ double s_coef[kMaxFields];
    const StepCtx sc = step_ctx(a);
    if (!APPLY && threadIdx.x == 0) load_coeffs(a, double(sc.step) * a.dt, s_coef);
    if (!APPLY) __syncthreads();

    const int P = a.n_s / VEC;
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= a.V * P) return;
    const int64_t i = a.row0 + tid / P;
    const int s0 = int(tid % P) * VEC;
    const int n_s = a.n_s;

    Upd<VEC> upd;
    if constexpr (!APPLY && PREF) upd_load<VEC>(a, sc, s_coef, i, s0, upd, true);

    double y[3][VEC];
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int v = 0; v < VEC; ++v) y[c][v] = 0.0;

    const int32_t l_end = __ldg(a.sym_lptr + i + 1);
#pragma unroll 2
    for (int32_t k = __ldg(a.sym_lptr + i); k < l_end; ++k) {          // blocks (i, j < i) = (j, i)^T
        const int64_t b = __ldg(a.sym_lidx + k);
        const int64_t j = __ldg(a.sym_lcol + k);
        const double* kp = a.Kval + b * 9 * n_s + s0;
        const double* up = sc.un + j * 3 * n_s + s0;
        Vec<VEC> u[3], kk[9];
#pragma unroll
        for (int d = 0; d < 3; ++d) u[d] = ld_ro<VEC>(up + d * n_s);
#pragma unroll
        for (int e = 0; e < 9; ++e) kk[e] = ld_once_l1<VEC>(kp + e * n_s);
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int d = 0; d < 3; ++d)
#pragma unroll
                for (int v = 0; v < VEC; ++v) y[c][v] = fma(kk[3 * d + c].v[v], u[d].v[v], y[c][v]);
    }
    const int2 ur = a.sym_urange[i];
#pragma unroll 2
    for (int32_t b = ur.x; b < ur.y; ++b) {                              // stored blocks (i, j >= i)
        const int64_t j = __ldg(a.sym_scol + b);
        const double* kp = a.Kval + int64_t(b) * 9 * n_s + s0;
        const double* up = sc.un + j * 3 * n_s + s0;
        Vec<VEC> u[3], kk[9];
#pragma unroll
        for (int d = 0; d < 3; ++d) u[d] = ld_ro<VEC>(up + d * n_s);
#pragma unroll
        for (int e = 0; e < 9; ++e) kk[e] = ld_once_l1<VEC>(kp + e * n_s);
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int d = 0; d < 3; ++d)
#pragma unroll
                for (int v = 0; v < VEC; ++v) y[c][v] = fma(kk[3 * c + d].v[v], u[d].v[v], y[c][v]);
    }
    if constexpr (APPLY) {
        store_y<VEC>(a, i, s0, y);
    } else {
        if constexpr (!PREF) upd_load<VEC>(a, sc, s_coef, i, s0, upd, true);
        upd_store<VEC>(a, sc, i, s0, y, upd);
    }
}

// ---- F2: fused step on the matrix-free element form ------------------------------------
// y[i][c][s] = sum over the incidences (e, a) of row i of alpha[e][s] * sum_{b, d}
//              K^_e[3a+c][3 loc(b) + d] u[node_b][d][s]
// Incidences are walked as fans around i (host_setup.cpp build_fans): incidence k uses the
// nodes (i, p_k, p_k+1) and the next one (i, p_k+1, p_k+2), so u[p_k+1] is loaded once and
// carried in registers.  The CTA's rows are contiguous, hence so are their incidences: one
// thread stages their K^ rows (224 B each) and fan records (16 B) into shared memory with
// two 1-D TMA bulk copies completing on an mbarrier, while every thread loads its own u_i.
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(bar), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    uint32_t done = 0;
    while (!done) {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done) : "r"(bar), "r"(phase) : "memory");
    }
}

template <int VEC>
__device__ __forceinline__ void cp_async_vec_s(uint32_t dst, const double* src) {
    if constexpr (VEC == 1) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" :: "r"(dst), "l"(src) : "memory");
    } else if constexpr (VEC == 2) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src) : "memory");
    } else {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst), "l"(src) : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" :: "r"(dst + 16), "l"(src + 2) : "memory");
    }
}

template <int VEC>
__device__ __forceinline__ Vec<VEC> lds_vec(const double* p) {
    Vec<VEC> r;
    if constexpr (VEC == 1) {
        r.v[0] = *p;
    } else if constexpr (VEC == 2) {
        const double2 t = *reinterpret_cast<const double2*>(p);
        r.v[0] = t.x; r.v[1] = t.y;
    } else {
        const double2 t0 = *reinterpret_cast<const double2*>(p), t1 = *reinterpret_cast<const double2*>(p + 2);
        r.v[0] = t0.x; r.v[1] = t0.y; r.v[2] = t1.x; r.v[3] = t1.y;
    }
    return r;
}

// ---- tile geometry shared by the matrix-free kernels ------------------------------------
// A tile = R consecutive rows (RCM order; launch ranges are R-aligned) x a chunk of
// W = G * VEC realisations.  Host-side lists give each row block its node set (own rows
// first, then every node its incidences reach) and element set; incidence records hold
// slots into those sets.
struct Tile {
    int64_t rb;          // global row-block index (= first row / R)
    int64_t r0;          // first row
    int nr;              // rows in the tile
    int32_t k0, n_inc;   // incidences [k0, k0 + n_inc)
    int32_t nd0, n_nodes, el0, n_els;
    int sbase, wv;       // realisation chunk
};

__device__ __forceinline__ Tile tile_of(const StepArgs& a, int64_t t, int64_t n_rb) {
    Tile T;
    const int R = a.mf_rows, W = a.mf_groups * 2;
    const int64_t chunk = t / n_rb;
    T.rb = a.row0 / R + (t - chunk * n_rb);
    T.r0 = T.rb * R;
    const int64_t r_end = a.row0 + a.V;
    T.nr = int((T.r0 + R < r_end ? T.r0 + R : r_end) - T.r0);
    T.k0 = __ldg(a.inc_ptr + T.r0);
    T.n_inc = __ldg(a.inc_ptr + T.r0 + T.nr) - T.k0;
    T.nd0 = __ldg(a.mf_node_ptr + T.rb);
    T.n_nodes = __ldg(a.mf_node_ptr + T.rb + 1) - T.nd0;
    T.el0 = __ldg(a.mf_el_ptr + T.rb);
    T.n_els = __ldg(a.mf_el_ptr + T.rb + 1) - T.el0;
    T.sbase = int(chunk) * W;
    T.wv = min(W, a.n_s - T.sbase);
    return T;
}

// One stage of the shared-memory ring (sizes from the per-launch maxima).
struct Stage {
    double* K;
    int4* rec;
    double* U;      // [nodes][3][W]
    double* A;      // [els][W]
    double* C;      // c1 [, c2, c3] of own rows: [1 or 3][R][W]
    double* O;      // u_{n-1} of own rows: [R][3][W]
};

__host__ __device__ __forceinline__ size_t stage_doubles(const StepArgs& a, bool c23) {
    const size_t W = size_t(a.mf_groups) * 2, R = size_t(a.mf_rows);
    return size_t(a.mf_smem_inc) * 30 + size_t(a.mf_nodes_max) * 3 * W + size_t(a.mf_els_max) * W +
           R * (c23 ? 3 : 1) * W + R * 3 * W;        // K 28 + rec 2 doubles per incidence
}

__device__ __forceinline__ Stage stage_at(const StepArgs& a, double* base, bool c23) {
    const int W = a.mf_groups * 2, R = a.mf_rows;
    Stage S;
    S.K = base;
    S.rec = reinterpret_cast<int4*>(S.K + size_t(a.mf_smem_inc) * 28);
    S.U = reinterpret_cast<double*>(S.rec + a.mf_smem_inc);
    S.A = S.U + size_t(a.mf_nodes_max) * 3 * W;
    S.C = S.A + size_t(a.mf_els_max) * W;
    S.O = S.C + size_t(R) * (c23 ? 3 : 1) * W;
    return S;
}

// Warp 0 stages tile T into S: lane 0 posts the byte count on the stage's mbarrier, then
// the lanes issue 1-D TMA bulk copies (every segment is a multiple of 16 B: N_s even).
template <bool APPLY>
__device__ __forceinline__ void stage_tile(const StepArgs& a, const StepCtx& sc, const Tile& T, const Stage& S,
                                           uint32_t bar, bool c23) {
    const int lane = int(threadIdx.x) & 31;
    const int W = a.mf_groups * 2, R = a.mf_rows, n_s = a.n_s;
    const bool full = T.wv == n_s;
    const uint32_t seg = uint32_t(T.wv) * 8u;
    if (lane == 0) {
        uint32_t tx = uint32_t(T.n_inc) * 240u + uint32_t(T.n_nodes * 3 + T.n_els) * seg;
        if (!APPLY) tx += uint32_t(T.nr) * seg * ((c23 ? 3u : 1u) + 3u);
        mbar_expect_tx(bar, tx);
        if (T.n_inc) {
            tma_bulk_g2s(uint32_t(__cvta_generic_to_shared(S.K)), a.Krow + size_t(T.k0) * 28, uint32_t(T.n_inc) * 224u, bar);
            tma_bulk_g2s(uint32_t(__cvta_generic_to_shared(S.rec)), a.fan + T.k0, uint32_t(T.n_inc) * 16u, bar);
        }
        if (!APPLY && full) {
            const int64_t r0 = T.r0;
            tma_bulk_g2s(uint32_t(__cvta_generic_to_shared(S.C)), a.c1 + r0 * n_s, uint32_t(T.nr) * seg, bar);
            if (c23) {
                tma_bulk_g2s(uint32_t(__cvta_generic_to_shared(S.C + size_t(R) * W)), a.c2a + r0 * n_s, uint32_t(T.nr) * seg, bar);
                tma_bulk_g2s(uint32_t(__cvta_generic_to_shared(S.C + size_t(2 * R) * W)), a.c3a + r0 * n_s, uint32_t(T.nr) * seg, bar);
            }
            tma_bulk_g2s(uint32_t(__cvta_generic_to_shared(S.O)), sc.uo + r0 * 3 * n_s, uint32_t(T.nr) * 3u * seg, bar);
        }
    }
    __syncwarp();
    for (int k = lane; k < T.n_nodes; k += 32) {
        const int64_t node = __ldg(a.mf_nodes + T.nd0 + k);
        const uint32_t dst = uint32_t(__cvta_generic_to_shared(S.U + size_t(k) * 3 * W));
        if (full) {
            tma_bulk_g2s(dst, sc.un + node * 3 * n_s, 3u * seg, bar);
        } else {
#pragma unroll
            for (int c = 0; c < 3; ++c)
                tma_bulk_g2s(dst + uint32_t(c * W * 8), sc.un + (node * 3 + c) * n_s + T.sbase, seg, bar);
        }
    }
    for (int k = lane; k < T.n_els; k += 32) {
        const int64_t e = __ldg(a.mf_els + T.el0 + k);
        tma_bulk_g2s(uint32_t(__cvta_generic_to_shared(S.A + size_t(k) * W)), a.alpha + e * n_s + T.sbase, seg, bar);
    }
    if (!APPLY && !full) {
        for (int r = lane; r < T.nr; r += 32) {
            const int64_t row = T.r0 + r;
            tma_bulk_g2s(uint32_t(__cvta_generic_to_shared(S.C + size_t(r) * W)), a.c1 + row * n_s + T.sbase, seg, bar);
            if (c23) {
                tma_bulk_g2s(uint32_t(__cvta_generic_to_shared(S.C + size_t(R + r) * W)), a.c2a + row * n_s + T.sbase, seg, bar);
                tma_bulk_g2s(uint32_t(__cvta_generic_to_shared(S.C + size_t(2 * R + r) * W)), a.c3a + row * n_s + T.sbase, seg, bar);
            }
#pragma unroll
            for (int c = 0; c < 3; ++c)
                tma_bulk_g2s(uint32_t(__cvta_generic_to_shared(S.O + (size_t(r) * 3 + c) * W)),
                             sc.uo + (row * 3 + c) * n_s + T.sbase, seg, bar);
        }
    }
}

constexpr int kMfThreads = 512;

// F2 (even N_s): persistent CTAs walk the tiles with a two-stage shared-memory ring.  While
// tile i is computed from stage i & 1, warp 0 has already issued the TMA copies of tile
// i + 1 into the other stage; one __syncthreads per tile frees a stage for reuse.  The
// gather and the update read only shared memory (plus F_k and the Dirichlet byte).
template <bool APPLY>
__global__ void __launch_bounds__(kMfThreads)
k_step_matrix_free_pipe(const StepArgs a) {
    constexpr int VEC = 2;
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ double s_coef[kMaxFields];
    __shared__ __align__(8) uint64_t s_full[2];

    const StepCtx sc = step_ctx(a);
    const bool c23 = a.c2a != nullptr;
    const int G = a.mf_groups, W = G * VEC, R = a.mf_rows, n_s = a.n_s;
    const int64_t n_rb = (a.V + R - 1) / R;
    const int64_t n_chunks = (n_s + W - 1) / W;
    const int64_t n_tiles = n_rb * n_chunks;
    const size_t sd = stage_doubles(a, c23);
    double* base = reinterpret_cast<double*>(smem);
    const uint32_t bar0 = uint32_t(__cvta_generic_to_shared(&s_full[0]));   // bar1 = bar0 + 8
    if (threadIdx.x == 0) {
        mbar_init(bar0, 1);
        mbar_init(bar0 + 8, 1);
        if (!APPLY) load_coeffs(a, double(sc.step) * a.dt, s_coef);
    }
    __syncthreads();
    int64_t t = blockIdx.x;
    if (t < n_tiles && threadIdx.x < 32) stage_tile<APPLY>(a, sc, tile_of(a, t, n_rb), stage_at(a, base, c23), bar0, c23);

    const int lr = int(threadIdx.x) / G, g = int(threadIdx.x) % G, w0 = g * VEC;
    for (int it = 0; t < n_tiles; ++it, t += gridDim.x) {
        const int st = it & 1;
        const int64_t tn = t + gridDim.x;
        if (tn < n_tiles && threadIdx.x < 32)
            stage_tile<APPLY>(a, sc, tile_of(a, tn, n_rb), stage_at(a, base + (st ^ 1) * sd, c23), bar0 + 8u * uint32_t(st ^ 1), c23);
        const Tile T = tile_of(a, t, n_rb);
        mbar_wait(bar0 + 8u * uint32_t(st), uint32_t(it >> 1) & 1u);
        const Stage X = stage_at(a, base + st * sd, c23);
        if (lr < T.nr && w0 < T.wv) {
            const int64_t i = T.r0 + lr;
            double y[3][VEC];
#pragma unroll
            for (int c = 0; c < 3; ++c)
#pragma unroll
                for (int v = 0; v < VEC; ++v) y[c][v] = 0.0;
            const double* Uw = X.U + w0;
            const double* Aw = X.A + w0;
            const int W3 = 3 * W;
            Vec<VEC> uo[3];
#pragma unroll
            for (int d = 0; d < 3; ++d) uo[d] = lds_vec<VEC>(Uw + lr * W3 + d * W);     // own row = slot lr
            const int32_t kb = __ldg(a.inc_ptr + i) - T.k0, ke = __ldg(a.inc_ptr + i + 1) - T.k0;
            for (int32_t k = kb; k < ke; ++k) {
                const int4 rec = X.rec[k];
                const double* K = X.K + k * 28;
                const double* Up = Uw + rec.y * W3;
                const double* Un = Uw + rec.z * W3;
                const Vec<VEC> al = lds_vec<VEC>(Aw + rec.x * W);
                double tt[3][VEC];
#pragma unroll
                for (int c = 0; c < 3; ++c)
#pragma unroll
                    for (int v = 0; v < VEC; ++v) tt[c][v] = 0.0;
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    const Vec<VEC> up = lds_vec<VEC>(Up + d * W), un = lds_vec<VEC>(Un + d * W);
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        const double k_own = K[9 * c + d], k_prev = K[9 * c + 3 + d], k_next = K[9 * c + 6 + d];
#pragma unroll
                        for (int v = 0; v < VEC; ++v) {
                            tt[c][v] = fma(k_own, uo[d].v[v], tt[c][v]);
                            tt[c][v] = fma(k_prev, up.v[v], tt[c][v]);
                            tt[c][v] = fma(k_next, un.v[v], tt[c][v]);
                        }
                    }
                }
#pragma unroll
                for (int c = 0; c < 3; ++c)
#pragma unroll
                    for (int v = 0; v < VEC; ++v) y[c][v] = fma(al.v[v], tt[c][v], y[c][v]);
            }
            const int s0 = T.sbase + w0;
            if constexpr (APPLY) {
                store_y<VEC>(a, i, s0, y);
            } else {
                Upd<VEC> u;
                u.fx = a.fixed ? __ldg(a.fixed + i) : uint8_t(0);
                u.c1 = lds_vec<VEC>(X.C + lr * W + w0);
                if (c23) {
                    u.c2 = lds_vec<VEC>(X.C + (R + lr) * W + w0);
                    u.c3 = lds_vec<VEC>(X.C + (2 * R + lr) * W + w0);
                } else {
#pragma unroll
                    for (int v = 0; v < VEC; ++v) { u.c2.v[v] = a.c2; u.c3.v[v] = a.c3; }
                }
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    u.un[c] = uo[c];
                    u.uo[c] = lds_vec<VEC>(X.O + lr * W3 + c * W + w0);
                    double f = 0.0;
                    for (int k = 0; k < a.n_fields; ++k) f = fma(s_coef[k], __ldg(a.Fk + (int64_t(k) * a.fk_rows + i) * 3 + c), f);
                    u.f[c] = f;
                }
                upd_store<VEC>(a, sc, i, s0, y, u);
            }
        }
        __syncthreads();                    // stage st is free for tile it + 2
    }
}

// F2 (odd N_s): direct gather from global memory, one thread per (row, realisation).
template <bool APPLY>
__global__ void __launch_bounds__(kThreads)
k_step_matrix_free_direct(const StepArgs a) {
    __shared__ double s_coef[kMaxFields];
    const StepCtx sc = step_ctx(a);
    if (!APPLY && threadIdx.x == 0) load_coeffs(a, double(sc.step) * a.dt, s_coef);
    if (!APPLY) __syncthreads();
    const int n_s = a.n_s;
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= a.V * n_s) return;
    const int64_t i = a.row0 + tid / n_s;
    const int s = int(tid % n_s);
    const int R = a.mf_rows;
    const int64_t rb = i / R;                            // records hold slots of the row block
    const int32_t nd0 = __ldg(a.mf_node_ptr + rb), el0 = __ldg(a.mf_el_ptr + rb);
    double y[3][1] = {{0.0}, {0.0}, {0.0}};
    double uo[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) uo[d] = __ldg(sc.un + (i * 3 + d) * n_s + s);
    for (int32_t k = __ldg(a.inc_ptr + i); k < __ldg(a.inc_ptr + i + 1); ++k) {
        const int4 rec = a.fan[k];
        const int64_t np = __ldg(a.mf_nodes + nd0 + rec.y), nn = __ldg(a.mf_nodes + nd0 + rec.z);
        const int64_t e = __ldg(a.mf_els + el0 + rec.x);
        const double* K = a.Krow + int64_t(k) * 28;
        const double al = __ldg(a.alpha + e * n_s + s);
        double tt[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const double up = __ldg(sc.un + (np * 3 + d) * n_s + s), un = __ldg(sc.un + (nn * 3 + d) * n_s + s);
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                tt[c] = fma(__ldg(K + 9 * c + d), uo[d], tt[c]);
                tt[c] = fma(__ldg(K + 9 * c + 3 + d), up, tt[c]);
                tt[c] = fma(__ldg(K + 9 * c + 6 + d), un, tt[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) y[c][0] = fma(al, tt[c], y[c][0]);
    }
    if constexpr (APPLY) {
        store_y<1>(a, i, s, y);
    } else {
        Upd<1> u;
        upd_load<1>(a, sc, s_coef, i, s, u, false);
#pragma unroll
        for (int c = 0; c < 3; ++c) u.un[c].v[0] = uo[c];
        upd_store<1>(a, sc, i, s, y, u);
    }
}

size_t mf_smem_bytes_impl(const StepArgs& a, int vec) {
    if (vec == 1) return 0;
    return 2 * stage_doubles(a, a.c2a != nullptr) * sizeof(double);
}

__global__ void k_advance(int64_t* step_base, int64_t n) { *step_base += n; }

// ---- F0: device assembly of the per-realisation block values ---------------------------
__global__ void __launch_bounds__(kThreads)
k_assemble(int64_t nnzb, int32_t n_s, const int32_t* __restrict__ cptr, const int32_t* __restrict__ contrib,
           const double* __restrict__ alpha, const double* __restrict__ Khat, double* __restrict__ Kval) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= nnzb * n_s) return;
    const int64_t b = tid / n_s;
    const int s = int(tid % n_s);
    double acc[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) acc[k] = 0.0;
    for (int32_t q = cptr[b]; q < cptr[b + 1]; ++q) {
        const int32_t code = contrib[q];
        const int64_t e = code / 9;
        const int ab = code % 9, la = ab / 3, lb = ab % 3;
        const double al = alpha[e * n_s + s];
        const double* K = Khat + e * 81;
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int d = 0; d < 3; ++d) acc[3 * c + d] = fma(al, K[9 * (3 * la + c) + 3 * lb + d], acc[3 * c + d]);
    }
#pragma unroll
    for (int k = 0; k < 9; ++k) Kval[(b * 9 + k) * n_s + s] = acc[k];
}

// ---- F4: layout transposes (ABI <-> device), off the hot path --------------------------
// device rows i < rows  <->  ABI [n_s][V_abi][3] at node map[i]
__global__ void k_abi_to_dev(int64_t rows, int32_t n_s, const int32_t* __restrict__ map, int64_t V_abi,
                             const double* __restrict__ src, double* __restrict__ dst) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= rows * 3 * n_s) return;
    const int s = int(tid % n_s);
    const int64_t ic = tid / n_s;
    const int64_t i = ic / 3;
    const int c = int(ic % 3);
    dst[tid] = src[(int64_t(s) * V_abi + map[i]) * 3 + c];
}

__global__ void k_dev_to_abi(int64_t rows, int32_t n_s, const int32_t* __restrict__ map, int64_t V_abi,
                             const double* __restrict__ src, double* __restrict__ dst) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (tid >= rows * 3 * n_s) return;
    const int s = int(tid % n_s);
    const int64_t ic = tid / n_s;
    const int64_t i = ic / 3;
    const int c = int(ic % 3);
    dst[(int64_t(s) * V_abi + map[i]) * 3 + c] = src[tid];
}

// ---- halo send-pack: sendbuf[k] = u_{n+1}[rows[k]] (3 n_s doubles per row) ------------
__global__ void k_pack(int64_t n, int32_t n_s, const int32_t* __restrict__ rows, const int64_t* step_base,
                       int64_t step_off, const double* ubuf0, const double* ubuf1, double* __restrict__ sendbuf) {
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t w = int64_t(3) * n_s;
    if (tid >= n * w) return;
    const int64_t step = *step_base + step_off;
    const double* unew = (step & 1) ? ubuf0 : ubuf1;     // u_{n+1} lives in buf[(step + 1) & 1]
    const int64_t k = tid / w;
    sendbuf[tid] = unew[int64_t(rows[k]) * w + (tid - k * w)];
}

inline unsigned grid_for(int64_t n) { return unsigned((n + kThreads - 1) / kThreads); }

}  // namespace


static bool a1_prefetch() {
    static int v = [] {
        const char* e = std::getenv("ENS_A1_PREFETCH");
        return e ? std::atoi(e) : 0;
    }();
    return v != 0;
}

template <int VEC, bool APPLY>
static cudaError_t launch_a1(const StepArgs& a, cudaStream_t st) {
    const int64_t n = a.V * (a.n_s / VEC);
    if (n == 0) return cudaSuccess;
    if (a1_prefetch()) k_step_assembled<VEC, APPLY, true><<<grid_for(n), kThreads, 0, st>>>(a);
    else k_step_assembled<VEC, APPLY, false><<<grid_for(n), kThreads, 0, st>>>(a);
    return cudaGetLastError();
}

template <bool APPLY>
static cudaError_t launch_a2_pipe(const StepArgs& a, cudaStream_t st) {
    if (a.V == 0) return cudaSuccess;
    const size_t smem = mf_smem_bytes_impl(a, 2);
    static int occ = -1;                 // CTAs per SM at this smem size (per instance)
    static size_t occ_smem = 0;
    if (occ < 0 || occ_smem != smem) {
        // dynamic + static shared memory must stay within the 227 KB per-CTA limit
        cudaError_t e = cudaFuncSetAttribute(k_step_matrix_free_pipe<APPLY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             int(smem));
        if (e != cudaSuccess) return e;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_step_matrix_free_pipe<APPLY>,
                                                          a.mf_rows * a.mf_groups, smem);
        if (e != cudaSuccess) return e;
        occ = occ < 1 ? 1 : occ;
        occ_smem = smem;
    }
    static int n_sm = 0;
    if (!n_sm) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    }
    const int P = a.n_s / 2;
    const int64_t n_tiles = ((a.V + a.mf_rows - 1) / a.mf_rows) * ((P + a.mf_groups - 1) / a.mf_groups);
    const int64_t grid = std::min<int64_t>(n_tiles, int64_t(n_sm) * occ);
    k_step_matrix_free_pipe<APPLY><<<unsigned(grid), unsigned(a.mf_rows * a.mf_groups), smem, st>>>(a);
    return cudaGetLastError();
}

template <bool APPLY>
static cudaError_t launch_a2_direct(const StepArgs& a, cudaStream_t st) {
    const int64_t n = a.V * a.n_s;
    if (n == 0) return cudaSuccess;
    k_step_matrix_free_direct<APPLY><<<grid_for(n), kThreads, 0, st>>>(a);
    return cudaGetLastError();
}

int pick_vec(int32_t n_s) {
    static int vec4 = [] {
        const char* e = std::getenv("ENS_A1_VEC4");
        return e ? std::atoi(e) : 0;
    }();
    if (vec4 && n_s % 4 == 0) return 4;
    return n_s % 2 == 0 ? 2 : 1;
}


template <int VEC, bool APPLY>
static cudaError_t launch_a1s(const StepArgs& a, cudaStream_t st) {
    const int64_t n = a.V * (a.n_s / VEC);
    if (n == 0) return cudaSuccess;
    if (a1_prefetch()) k_step_assembled_sym<VEC, APPLY, true><<<grid_for(n), kThreads, 0, st>>>(a);
    else k_step_assembled_sym<VEC, APPLY, false><<<grid_for(n), kThreads, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_step_assembled_sym(const StepArgs& a, cudaStream_t st) {
    const bool apply = a.y_out != nullptr;
    switch (pick_vec(a.n_s)) {
        case 4: return apply ? launch_a1s<4, true>(a, st) : launch_a1s<4, false>(a, st);
        case 2: return apply ? launch_a1s<2, true>(a, st) : launch_a1s<2, false>(a, st);
        default: return apply ? launch_a1s<1, true>(a, st) : launch_a1s<1, false>(a, st);
    }
}

cudaError_t launch_step_assembled(const StepArgs& a, cudaStream_t st) {
    const bool apply = a.y_out != nullptr;
    switch (pick_vec(a.n_s)) {
        case 4: return apply ? launch_a1<4, true>(a, st) : launch_a1<4, false>(a, st);
        case 2: return apply ? launch_a1<2, true>(a, st) : launch_a1<2, false>(a, st);
        default: return apply ? launch_a1<1, true>(a, st) : launch_a1<1, false>(a, st);
    }
}

int pick_vec_mf(int32_t n_s) { return n_s % 2 ? 1 : 2; }

size_t mf_smem_bytes(const StepArgs& a, int vec) { return mf_smem_bytes_impl(a, vec); }

cudaError_t launch_step_matrix_free(const StepArgs& a, cudaStream_t st) {
    const bool ap = a.y_out != nullptr;
    if (pick_vec_mf(a.n_s) == 2) return ap ? launch_a2_pipe<true>(a, st) : launch_a2_pipe<false>(a, st);
    return ap ? launch_a2_direct<true>(a, st) : launch_a2_direct<false>(a, st);
}

cudaError_t launch_advance(int64_t* step_base, int64_t n, cudaStream_t st) {
    k_advance<<<1, 1, 0, st>>>(step_base, n);
    return cudaGetLastError();
}

cudaError_t launch_assemble(int64_t nnzb, int32_t n_s, const int32_t* contrib_ptr, const int32_t* contrib,
                            const double* alpha, const double* Khat, double* Kval, cudaStream_t st) {
    const int64_t n = nnzb * n_s;
    if (n == 0) return cudaSuccess;
    k_assemble<<<grid_for(n), kThreads, 0, st>>>(nnzb, n_s, contrib_ptr, contrib, alpha, Khat, Kval);
    return cudaGetLastError();
}

cudaError_t launch_abi_to_dev(int64_t rows, int32_t n_s, const int32_t* map, int64_t V_abi, const double* src,
                              double* dst, cudaStream_t st) {
    const int64_t n = rows * 3 * n_s;
    if (n == 0) return cudaSuccess;
    k_abi_to_dev<<<grid_for(n), kThreads, 0, st>>>(rows, n_s, map, V_abi, src, dst);
    return cudaGetLastError();
}

cudaError_t launch_dev_to_abi(int64_t rows, int32_t n_s, const int32_t* map, int64_t V_abi, const double* src,
                              double* dst, cudaStream_t st) {
    const int64_t n = rows * 3 * n_s;
    if (n == 0) return cudaSuccess;
    k_dev_to_abi<<<grid_for(n), kThreads, 0, st>>>(rows, n_s, map, V_abi, src, dst);
    return cudaGetLastError();
}

cudaError_t launch_pack(int64_t n, int32_t n_s, const int32_t* rows, const int64_t* step_base, int64_t step_off,
                        const double* ubuf0, const double* ubuf1, double* sendbuf, cudaStream_t st) {
    const int64_t m = n * 3 * n_s;
    if (m == 0) return cudaSuccess;
    k_pack<<<grid_for(m), kThreads, 0, st>>>(n, n_s, rows, step_base, step_off, ubuf0, ubuf1, sendbuf);
    return cudaGetLastError();
}

}  // namespace ens
