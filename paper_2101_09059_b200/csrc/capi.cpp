// capi.cpp -- the C ABI of include/ens.h: context lifetime, host setup -> device upload,
// step enqueue, state transfer.  Every step of the hot path runs in kernels.cu.
#include "ens.h"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "device.hpp"
#include "host_setup.hpp"

namespace {

thread_local std::string g_err;

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

}  // namespace

struct ens_ctx {
    std::string err;
    int device = 0;
    cudaStream_t stream = nullptr;
    void* (*dev_alloc)(size_t, void*) = nullptr;
    void (*dev_free)(void*, void*) = nullptr;
    void* alloc_user = nullptr;
    std::vector<DevBuf> bufs;
    int64_t device_bytes = 0;

    int64_t V = 0, F = 0, nnzb = 0;
    int32_t n_s = 0, s_begin = 0;
    int32_t kernel = 0, damping = 0, dist = 0;
    double dt = 0.0, dt_cfl = 0.0, c_d = 0.0;
    int32_t bandwidth = 0;
    std::vector<int32_t> perm, iperm;      // perm[new] = old

    // device arrays (RCM order, realisation innermost)
    int32_t *d_row_ptr = nullptr, *d_col = nullptr, *d_perm = nullptr;
    double *d_Kval = nullptr, *d_c1 = nullptr, *d_c2a = nullptr, *d_c3a = nullptr;
    double c2 = 2.0, c3 = 1.0;
    uint8_t* d_fixed = nullptr;
    int32_t* d_inc_ptr = nullptr;
    int4* d_fan = nullptr;
    double *d_Krow = nullptr, *d_Khat = nullptr, *d_alpha = nullptr;
    int32_t mf_rows = 1, mf_groups = 1, mf_smem_inc = 0;
    double *d_u0 = nullptr, *d_u1 = nullptr, *d_stage = nullptr;
    double *d_scratch_u = nullptr, *d_scratch_y = nullptr;
    unsigned long long* d_flag = nullptr;
    int64_t* d_step = nullptr;
    // traction
    int32_t n_fields = 0, n_tab = 0;
    double *d_Fk = nullptr, *d_tab_t = nullptr, *d_tab_g = nullptr;
    double period = 0.0, ramp_T = 0.0;

    int64_t step = 0;       // host mirror of *d_step once the stream drains
    bool latched = false;

    // CUDA graph of graph_steps fused steps + one counter advance, replayed by ens_step
    int32_t graph_steps = 64;
    cudaGraphExec_t graph = nullptr;
    bool graph_dirty = true;
};

namespace {

int fail(ens_ctx* c, int code, const std::string& msg) {
    g_err = msg;
    if (c) c->err = msg;
    return code;
}

int cuda_fail(ens_ctx* c, cudaError_t e, const char* what) {
    return fail(c, e == cudaErrorMemoryAllocation ? ENS_E_OOM : ENS_E_CUDA,
                std::string(what) + ": " + cudaGetErrorString(e));
}

#define CUDA_TRY(c, expr)                                   \
    do {                                                    \
        cudaError_t _e = (expr);                            \
        if (_e != cudaSuccess) return cuda_fail(c, _e, #expr); \
    } while (0)

template <typename T>
int dalloc(ens_ctx* c, T** out, size_t count) {
    *out = nullptr;
    size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    void* p = nullptr;
    if (c->dev_alloc) {
        p = c->dev_alloc(bytes, c->alloc_user);
        if (!p) return fail(c, ENS_E_OOM, "device allocation of " + std::to_string(bytes) + " bytes failed");
    } else {
        cudaError_t e = cudaMallocAsync(&p, bytes, c->stream);
        if (e != cudaSuccess) return cuda_fail(c, e, "cudaMallocAsync");
    }
    c->bufs.push_back({p, bytes});
    c->device_bytes += int64_t(bytes);
    *out = static_cast<T*>(p);
    return ENS_OK;
}

template <typename T>
void dfree(ens_ctx* c, T*& p) {
    if (!p) return;
    for (size_t k = 0; k < c->bufs.size(); ++k)
        if (c->bufs[k].p == static_cast<void*>(p)) {
            if (c->dev_free) c->dev_free(c->bufs[k].p, c->alloc_user);
            else cudaFreeAsync(c->bufs[k].p, c->stream);
            c->device_bytes -= int64_t(c->bufs[k].bytes);
            c->bufs.erase(c->bufs.begin() + int64_t(k));
            break;
        }
    p = nullptr;
}

template <typename T>
int upload(ens_ctx* c, T** out, const T* host, size_t count) {
    int rc = dalloc(c, out, count);
    if (rc) return rc;
    if (count) CUDA_TRY(c, cudaMemcpyAsync(*out, host, count * sizeof(T), cudaMemcpyHostToDevice, c->stream));
    // host staging vectors die at the end of ens_create: make the copy complete first
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return ENS_OK;
}

void free_all(ens_ctx* c) {
    if (c->stream) cudaStreamSynchronize(c->stream);
    for (auto& b : c->bufs) {
        if (c->dev_free) c->dev_free(b.p, c->alloc_user);
        else cudaFreeAsync(b.p, c->stream);
    }
    if (c->stream) cudaStreamSynchronize(c->stream);
    c->bufs.clear();
}

int check_opts(const ens_options* opt) {
    if (!opt) return ENS_OK;
    if (!(std::isfinite(opt->dt))) return fail(nullptr, ENS_E_ARG, "opt->dt is not finite");
    if (opt->damping < 0 || opt->damping > 2) return fail(nullptr, ENS_E_ARG, "opt->damping must be 0, 1 or 2");
    if (opt->kernel < 0 || opt->kernel > 1) return fail(nullptr, ENS_E_ARG, "opt->kernel must be 0 or 1");
    if (!(opt->c_d >= 0.0) || !std::isfinite(opt->c_d)) return fail(nullptr, ENS_E_ARG, "opt->c_d must be finite and >= 0");
    if (opt->dist == ENS_DIST_NODE)
        return fail(nullptr, ENS_E_UNSUPPORTED, "dist = ENS_DIST_NODE is not built in this version (use ENS_DIST_ENSEMBLE)");
    if (opt->dist < 0 || opt->dist > 2) return fail(nullptr, ENS_E_ARG, "opt->dist must be 0, 1 or 2");
    return ENS_OK;
}

int init_ctx(ens_ctx* c, const ens_options* opt) {
    ens_options def{};
    if (!opt) opt = &def;
    c->device = opt->device;
    if (opt->device >= 0) CUDA_TRY(c, cudaSetDevice(opt->device));
    else CUDA_TRY(c, cudaGetDevice(&c->device));
    c->stream = static_cast<cudaStream_t>(opt->stream);
    c->dev_alloc = opt->dev_alloc;
    c->dev_free = opt->dev_free;
    c->alloc_user = opt->alloc_user;
    c->kernel = opt->kernel;
    c->damping = opt->damping;
    c->dist = opt->dist;
    c->c_d = opt->c_d;
    return ENS_OK;
}

int alloc_state(ens_ctx* c) {
    const size_t n = size_t(c->V) * 3 * size_t(c->n_s);
    int rc;
    if ((rc = dalloc(c, &c->d_u0, n)) || (rc = dalloc(c, &c->d_u1, n)) || (rc = dalloc(c, &c->d_stage, n)) ||
        (rc = dalloc(c, &c->d_flag, 1)) || (rc = dalloc(c, &c->d_step, 1)))
        return rc;
    CUDA_TRY(c, cudaMemsetAsync(c->d_u0, 0, n * sizeof(double), c->stream));
    CUDA_TRY(c, cudaMemsetAsync(c->d_u1, 0, n * sizeof(double), c->stream));
    CUDA_TRY(c, cudaMemsetAsync(c->d_flag, 0xff, sizeof(unsigned long long), c->stream));
    CUDA_TRY(c, cudaMemsetAsync(c->d_step, 0, sizeof(int64_t), c->stream));
    c->step = 0;
    return ENS_OK;
}

ens::StepArgs step_args(const ens_ctx* c) {
    ens::StepArgs a;
    a.V = c->V;
    a.row0 = 0;
    a.V_total = c->V;
    a.n_s = c->n_s;
    a.row_ptr = c->d_row_ptr;
    a.col = c->d_col;
    a.Kval = c->d_Kval;
    a.inc_ptr = c->d_inc_ptr;
    a.fan = c->d_fan;
    a.Krow = c->d_Krow;
    a.alpha = c->d_alpha;
    a.mf_rows = c->mf_rows;
    a.mf_groups = c->mf_groups;
    a.mf_smem_inc = c->mf_smem_inc;
    a.c1 = c->d_c1;
    a.c2a = c->d_c2a;
    a.c3a = c->d_c3a;
    a.c2 = c->c2;
    a.c3 = c->c3;
    a.fixed = c->d_fixed;
    a.n_fields = c->n_fields;
    a.Fk = c->d_Fk;
    a.n_tab = c->n_tab;
    a.tab_t = c->d_tab_t;
    a.tab_g = c->d_tab_g;
    a.period = c->period;
    a.ramp_T = c->ramp_T;
    a.dt = c->dt;
    a.step_base = c->d_step;
    a.ubuf0 = c->d_u0;
    a.ubuf1 = c->d_u1;
    a.flag = c->d_flag;
    a.s_global0 = c->s_begin;
    return a;
}

cudaError_t launch(const ens_ctx* c, const ens::StepArgs& a) {
    return c->kernel == ENS_KERNEL_MATRIX_FREE ? ens::launch_step_matrix_free(a, c->stream)
                                               : ens::launch_step_assembled(a, c->stream);
}

// Element -> node-block contributions for F0, ascending element within each block.
int build_device_operator(ens_ctx* c, const ens::MeshView& m, const ens::Pattern& pat,
                          const std::vector<double>& Khat, const std::vector<double>& alpha_se) {
    const int64_t F = c->F, n_s = c->n_s;
    // alpha in device layout [F][n_s]
    std::vector<double> alpha_dev(size_t(F * n_s));
    for (int64_t s = 0; s < n_s; ++s)
        for (int64_t e = 0; e < F; ++e) alpha_dev[size_t(e * n_s + s)] = alpha_se[size_t(s * F + e)];
    int rc;
    if ((rc = upload(c, &c->d_alpha, alpha_dev.data(), alpha_dev.size()))) return rc;
    if ((rc = upload(c, &c->d_Khat, Khat.data(), Khat.size()))) return rc;

    if (c->kernel == ENS_KERNEL_ASSEMBLED) {
        std::vector<int32_t> cnt(size_t(c->nnzb) + 1, 0), code(size_t(9 * F)), blk(size_t(9 * F));
        for (int64_t e = 0; e < F; ++e)
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) {
                    int32_t i = pat.iperm[size_t(m.tris[3 * e + a])], j = pat.iperm[size_t(m.tris[3 * e + b])];
                    auto first = pat.col.begin() + pat.row_ptr[size_t(i)];
                    auto last = pat.col.begin() + pat.row_ptr[size_t(i) + 1];
                    auto it = std::lower_bound(first, last, j);
                    int32_t bi = int32_t(it - pat.col.begin());
                    blk[size_t(9 * e + 3 * a + b)] = bi;
                    cnt[size_t(bi) + 1]++;
                }
        for (size_t k = 1; k < cnt.size(); ++k) cnt[k] += cnt[k - 1];
        std::vector<int32_t> fillp(cnt.begin(), cnt.end() - 1);
        for (int64_t e = 0; e < F; ++e)                 // ascending e => ascending within block
            for (int ab = 0; ab < 9; ++ab) code[size_t(fillp[size_t(blk[size_t(9 * e + ab)])]++)] = int32_t(9 * e + ab);
        int32_t *d_cptr = nullptr, *d_code = nullptr;
        if ((rc = upload(c, &d_cptr, cnt.data(), cnt.size())) || (rc = upload(c, &d_code, code.data(), code.size())))
            return rc;
        if ((rc = dalloc(c, &c->d_Kval, size_t(c->nnzb) * 9 * size_t(n_s)))) return rc;
        CUDA_TRY(c, ens::launch_assemble(c->nnzb, c->n_s, d_cptr, d_code, c->d_alpha, c->d_Khat, c->d_Kval, c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        dfree(c, d_cptr);
        dfree(c, d_code);
        dfree(c, c->d_alpha);       // the assembled path needs only Kval from here on
        dfree(c, c->d_Khat);
    } else {
        ens::Fans fans = ens::build_fans(m, pat.iperm, Khat);
        dfree(c, c->d_Khat);                      // Krow holds K^ in gather order
        // CTA geometry: G threads per row (one realisation group each), R rows per CTA
        const int P = c->n_s / ens::pick_vec(c->n_s);
        c->mf_groups = std::min(P, 256);
        c->mf_rows = std::max(1, std::min(256 / c->mf_groups, 32));
        for (;;) {
            int32_t mx = 0;
            for (int64_t r0 = 0; r0 < c->V; r0 += c->mf_rows) {
                int64_t r1 = std::min<int64_t>(r0 + c->mf_rows, c->V);
                mx = std::max(mx, fans.ptr[size_t(r1)] - fans.ptr[size_t(r0)]);
            }
            c->mf_smem_inc = mx;
            if (int64_t(mx) * 240 <= 96 * 1024 || c->mf_rows == 1) break;
            c->mf_rows = std::max(1, c->mf_rows / 2);
        }
        if (int64_t(c->mf_smem_inc) * 240 > 200 * 1024)
            return fail(c, ENS_E_UNSUPPORTED, "a node has too many incident elements for the matrix-free kernel");
        static_assert(sizeof(ens::FanRec) == sizeof(int4), "FanRec layout");
        if ((rc = upload(c, &c->d_inc_ptr, fans.ptr.data(), fans.ptr.size())) ||
            (rc = upload(c, &c->d_fan, reinterpret_cast<const int4*>(fans.rec.data()), fans.rec.size())) ||
            (rc = upload(c, &c->d_Krow, fans.Krow.data(), fans.Krow.size())))
            return rc;
    }
    return ENS_OK;
}

int finish_create(ens_ctx* c, ens_ctx** out) {
    int rc = alloc_state(c);
    if (rc) return rc;
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (const char* g = std::getenv("ENS_GRAPH_STEPS")) c->graph_steps = std::max(0, std::atoi(g));
    *out = c;
    return ENS_OK;
}

void drop_graph(ens_ctx* c) {
    if (c->graph) cudaGraphExecDestroy(c->graph);
    c->graph = nullptr;
    c->graph_dirty = true;
}

// Capture graph_steps launches (step_off = 0..G-1) + the counter advance on a private
// stream (the caller's stream may be the legacy default stream, which cannot capture).
int build_graph(ens_ctx* c) {
    drop_graph(c);
    cudaStream_t cap = nullptr;
    CUDA_TRY(c, cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    ens::StepArgs a = step_args(c);
    cudaError_t err = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    for (int32_t k = 0; err == cudaSuccess && k < c->graph_steps; ++k) {
        a.step_off = k;
        err = c->kernel == ENS_KERNEL_MATRIX_FREE ? ens::launch_step_matrix_free(a, cap)
                                                  : ens::launch_step_assembled(a, cap);
    }
    if (err == cudaSuccess) err = ens::launch_advance(c->d_step, c->graph_steps, cap);
    cudaGraph_t g = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(cap, &g);
    if (err == cudaSuccess) err = e2;
    if (err == cudaSuccess) err = cudaGraphInstantiate(&c->graph, g, 0);
    if (g) cudaGraphDestroy(g);
    cudaStreamDestroy(cap);
    if (err != cudaSuccess) return cuda_fail(c, err, "CUDA graph capture of the step loop");
    c->graph_dirty = false;
    return ENS_OK;
}

}  // namespace

extern "C" {

int ens_create(const ens_mesh* mesh, const ens_materials* mat, const ens_options* opt, ens_ctx** out) {
    if (!out) return fail(nullptr, ENS_E_ARG, "out is NULL");
    *out = nullptr;
    if (!mesh || !mat) return fail(nullptr, ENS_E_ARG, "mesh or materials is NULL");
    if (mesh->n_nodes < 1 || mesh->n_tris < 1 || !mesh->xyz || !mesh->tris)
        return fail(nullptr, ENS_E_ARG, "mesh needs n_nodes >= 1, n_tris >= 1, xyz and tris");
    if (mesh->n_nodes >= (int64_t(1) << 31) || 3 * mesh->n_tris >= (int64_t(1) << 31))
        return fail(nullptr, ENS_E_ARG, "mesh too large for 32-bit node / element ids");
    if (mat->n_s < 1 || !mat->E || !mat->h) return fail(nullptr, ENS_E_ARG, "materials need n_s >= 1, E and h");
    if (!(mat->rho > 0.0) || !std::isfinite(mat->rho)) return fail(nullptr, ENS_E_ARG, "rho must be > 0");
    if (!(mat->nu >= 0.0 && mat->nu <= 0.5)) return fail(nullptr, ENS_E_ARG, "nu must lie in [0, 0.5]");
    if (!(mat->k_shear > 0.0) || !std::isfinite(mat->k_shear)) return fail(nullptr, ENS_E_ARG, "k_shear must be > 0");
    int rc = check_opts(opt);
    if (rc) return rc;
    const int64_t V = mesh->n_nodes, F = mesh->n_tris, NV = int64_t(mat->n_s) * V;
    for (int64_t k = 0; k < NV; ++k) {
        if (!(mat->E[k] > 0.0) || !std::isfinite(mat->E[k]))
            return fail(nullptr, ENS_E_ARG, "E[" + std::to_string(k / V) + "][" + std::to_string(k % V) + "] must be finite and > 0");
        if (!(mat->h[k] > 0.0) || !std::isfinite(mat->h[k]))
            return fail(nullptr, ENS_E_ARG, "h[" + std::to_string(k / V) + "][" + std::to_string(k % V) + "] must be finite and > 0");
    }
    ens::MeshView m{V, F, mesh->xyz, mesh->tris};
    int64_t bad = -1;
    int vcode = ens::validate_mesh(m, &bad);
    if (vcode) {
        static const char* what[] = {"", "node index out of range in element ", "repeated node in element ",
                                     "degenerate (zero-area) element ", "edge shared by more than two triangles at node "};
        return fail(nullptr, ENS_E_MESH, std::string(what[vcode]) + std::to_string(bad));
    }

    ens_ctx* c = new ens_ctx();
    if ((rc = init_ctx(c, opt))) { delete c; return rc; }
    c->V = V;
    c->F = F;
    c->n_s = mat->n_s;
    c->s_begin = mat->s_begin;

    // S0: pattern (RCM + block CSR)
    ens::Pattern pat = ens::build_pattern(m);
    c->nnzb = int64_t(pat.col.size());
    c->bandwidth = pat.bandwidth;
    c->perm = pat.perm;
    c->iperm = pat.iperm;
    if (c->nnzb >= (int64_t(1) << 31)) { delete c; return fail(nullptr, ENS_E_ARG, "pattern exceeds 2^31 blocks"); }

    // S1: element stiffness, Gauss-point scaling, mass, CFL, coefficients
    std::vector<double> Khat(size_t(81 * F)), area(static_cast<size_t>(F));
    for (int64_t e = 0; e < F; ++e)
        ens::element_stiffness(mesh->xyz + 3 * int64_t(mesh->tris[3 * e]), mesh->xyz + 3 * int64_t(mesh->tris[3 * e + 1]),
                               mesh->xyz + 3 * int64_t(mesh->tris[3 * e + 2]), mat->nu, mat->k_shear,
                               Khat.data() + 81 * e, area.data() + e);
    std::vector<double> alpha(size_t(mat->n_s * F)), mass(static_cast<size_t>(NV));
    ens::materials(m, mat->n_s, mat->E, mat->h, mat->rho, alpha.data(), mass.data());
    double safety = (opt && opt->cfl_safety > 0.0) ? opt->cfl_safety : 0.9;
    c->dt_cfl = ens::cfl_dt(m, mat->n_s, mat->E, mat->rho, safety);
    c->dt = (opt && opt->dt > 0.0) ? opt->dt : c->dt_cfl;

    const int64_t n_s = c->n_s;
    const double dt = c->dt;
    std::vector<double> c1(static_cast<size_t>(NV)), c2a, c3a;
    if (c->damping == ENS_DAMP_IDENTITY) { c2a.resize(size_t(NV)); c3a.resize(size_t(NV)); }
    for (int64_t i = 0; i < V; ++i)
        for (int64_t s = 0; s < n_s; ++s) {
            const double mi = mass[size_t(s * V + pat.perm[size_t(i)])];
            double cc = c->damping == ENS_DAMP_MASS ? c->c_d * mi : (c->damping == ENS_DAMP_IDENTITY ? c->c_d : 0.0);
            double D = mi + 0.5 * dt * cc;
            c1[size_t(i * n_s + s)] = dt * dt / D;
            if (c->damping == ENS_DAMP_IDENTITY) {
                c2a[size_t(i * n_s + s)] = 2.0 * mi / D;
                c3a[size_t(i * n_s + s)] = (mi - 0.5 * dt * cc) / D;
            }
        }
    if (c->damping == ENS_DAMP_MASS) {      // C~ = c_d M~: c2, c3 independent of the node
        double q = 0.5 * dt * c->c_d;
        c->c2 = 2.0 / (1.0 + q);
        c->c3 = (1.0 - q) / (1.0 + q);
    }
    std::vector<int32_t> rp32(pat.row_ptr.begin(), pat.row_ptr.end());
    std::vector<uint8_t> fixed(size_t(V), 0);
    if (mesh->fixed)
        for (int64_t i = 0; i < V; ++i) fixed[size_t(i)] = mesh->fixed[pat.perm[size_t(i)]] & 7;

    if ((rc = upload(c, &c->d_row_ptr, rp32.data(), rp32.size())) || (rc = upload(c, &c->d_col, pat.col.data(), pat.col.size())) ||
        (rc = upload(c, &c->d_perm, pat.perm.data(), pat.perm.size())) || (rc = upload(c, &c->d_fixed, fixed.data(), fixed.size())) ||
        (rc = upload(c, &c->d_c1, c1.data(), c1.size())) ||
        (c->damping == ENS_DAMP_IDENTITY && ((rc = upload(c, &c->d_c2a, c2a.data(), c2a.size())) ||
                                            (rc = upload(c, &c->d_c3a, c3a.data(), c3a.size())))) ||
        (rc = build_device_operator(c, m, pat, Khat, alpha)) || (rc = finish_create(c, out))) {
        std::string msg = c->err;
        free_all(c);
        delete c;
        g_err = msg;
        return rc;
    }
    return ENS_OK;
}

int ens_create_csr(int64_t n_nodes, const int64_t* row_ptr, const int32_t* col, int32_t n_s, const double* Kval,
                   const double* c1, const double* c2, const double* c3, const uint8_t* fixed, double dt,
                   const ens_options* opt, ens_ctx** out) {
    if (!out) return fail(nullptr, ENS_E_ARG, "out is NULL");
    *out = nullptr;
    if (n_nodes < 1 || !row_ptr || !col || n_s < 1 || !Kval || !c1 || !c2 || !c3)
        return fail(nullptr, ENS_E_ARG, "ens_create_csr: bad arguments");
    int rc = check_opts(opt);
    if (rc) return rc;
    if (opt && opt->kernel != ENS_KERNEL_ASSEMBLED) return fail(nullptr, ENS_E_ARG, "ens_create_csr needs kernel = ASSEMBLED");
    const int64_t V = n_nodes, nnzb = row_ptr[V];
    for (int64_t i = 0; i < V; ++i)
        if (row_ptr[i + 1] < row_ptr[i]) return fail(nullptr, ENS_E_ARG, "row_ptr not monotone");
    for (int64_t b = 0; b < nnzb; ++b)
        if (col[b] < 0 || col[b] >= V) return fail(nullptr, ENS_E_ARG, "column index out of range");
    ens_ctx* c = new ens_ctx();
    if ((rc = init_ctx(c, opt))) { delete c; return rc; }
    c->kernel = ENS_KERNEL_ASSEMBLED;
    c->damping = ENS_DAMP_IDENTITY;          // arbitrary per-DOF c2, c3 arrays
    c->V = V;
    c->F = 0;
    c->nnzb = nnzb;
    c->n_s = n_s;
    c->dt = c->dt_cfl = dt;
    c->perm.resize(size_t(V));
    for (int64_t i = 0; i < V; ++i) c->perm[size_t(i)] = int32_t(i);
    c->iperm = c->perm;
    // caller layout -> device layout
    std::vector<double> kv(size_t(nnzb * 9 * n_s)), a1(size_t(V * n_s)), a2(a1.size()), a3(a1.size());
    for (int64_t s = 0; s < n_s; ++s) {
        for (int64_t b = 0; b < nnzb; ++b)
            for (int k = 0; k < 9; ++k) kv[size_t((b * 9 + k) * n_s + s)] = Kval[(s * nnzb + b) * 9 + k];
        for (int64_t i = 0; i < V; ++i) {
            a1[size_t(i * n_s + s)] = c1[s * V + i];
            a2[size_t(i * n_s + s)] = c2[s * V + i];
            a3[size_t(i * n_s + s)] = c3[s * V + i];
        }
    }
    std::vector<int32_t> rp32(row_ptr, row_ptr + V + 1);
    std::vector<uint8_t> fx(size_t(V), 0);
    if (fixed)
        for (int64_t i = 0; i < V; ++i) fx[size_t(i)] = fixed[i] & 7;
    if ((rc = upload(c, &c->d_row_ptr, rp32.data(), rp32.size())) || (rc = upload(c, &c->d_col, col, size_t(nnzb))) ||
        (rc = upload(c, &c->d_perm, c->perm.data(), c->perm.size())) || (rc = upload(c, &c->d_fixed, fx.data(), fx.size())) ||
        (rc = upload(c, &c->d_Kval, kv.data(), kv.size())) || (rc = upload(c, &c->d_c1, a1.data(), a1.size())) ||
        (rc = upload(c, &c->d_c2a, a2.data(), a2.size())) || (rc = upload(c, &c->d_c3a, a3.data(), a3.size())) ||
        (rc = finish_create(c, out))) {
        std::string msg = c->err;
        free_all(c);
        delete c;
        g_err = msg;
        return rc;
    }
    return ENS_OK;
}

int ens_set_traction(ens_ctx* c, int32_t n_fields, const double* F, int32_t n_tab, const double* tab_t,
                     const double* tab_g, double period, double ramp_T) {
    if (!c) return fail(nullptr, ENS_E_ARG, "ctx is NULL");
    if (n_fields < 0 || n_fields > ens::kMaxFields) return fail(c, ENS_E_ARG, "n_fields must be in [0, 4]");
    if (n_fields > 0 && !F) return fail(c, ENS_E_ARG, "F is NULL");
    if (n_tab < 0 || (n_tab > 0 && (!tab_t || !tab_g))) return fail(c, ENS_E_ARG, "bad table");
    for (int32_t k = 0; k + 1 < n_tab; ++k)
        if (!(tab_t[k] < tab_t[k + 1])) return fail(c, ENS_E_ARG, "tab_t must be strictly increasing");
    if (!std::isfinite(period) || !std::isfinite(ramp_T)) return fail(c, ENS_E_ARG, "period / ramp_T not finite");
    const int64_t V = c->V;
    std::vector<double> Fd(size_t(n_fields * V * 3));
    for (int32_t k = 0; k < n_fields; ++k)
        for (int64_t i = 0; i < V; ++i)
            for (int d = 0; d < 3; ++d) Fd[size_t((k * V + i) * 3 + d)] = F[(k * V + c->perm[size_t(i)]) * 3 + d];
    // (re)allocate: sizes may change; keep previous buffers alive until the stream drains
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    drop_graph(c);
    dfree(c, c->d_Fk);
    dfree(c, c->d_tab_t);
    dfree(c, c->d_tab_g);
    c->n_fields = 0;
    c->n_tab = 0;
    int rc;
    if ((rc = upload(c, &c->d_Fk, Fd.data(), Fd.size()))) return rc;
    if (n_tab > 0) {
        if ((rc = upload(c, &c->d_tab_t, tab_t, size_t(n_tab))) || (rc = upload(c, &c->d_tab_g, tab_g, size_t(n_tab) * n_fields)))
            return rc;
    }
    c->n_fields = n_fields;
    c->n_tab = n_tab;
    c->period = period;
    c->ramp_T = ramp_T;
    return ENS_OK;
}

int ens_step(ens_ctx* c, int64_t n) {
    if (!c) return fail(nullptr, ENS_E_ARG, "ctx is NULL");
    if (n < 0) return fail(c, ENS_E_ARG, "n must be >= 0");
    if (c->latched) return fail(c, ENS_E_STATE, "context diverged: call ens_set_state before stepping again");
    int64_t left = n;
    if (c->graph_steps > 0 && n >= c->graph_steps) {
        if (c->graph_dirty) {
            int rc = build_graph(c);
            if (rc) return rc;
        }
        for (; left >= c->graph_steps; left -= c->graph_steps) CUDA_TRY(c, cudaGraphLaunch(c->graph, c->stream));
    }
    ens::StepArgs a = step_args(c);
    for (int64_t k = 0; k < left; ++k) {
        a.step_off = k;
        CUDA_TRY(c, launch(c, a));
    }
    if (left) CUDA_TRY(c, ens::launch_advance(c->d_step, left, c->stream));
    c->step += n;
    return ENS_OK;
}

int ens_sync(ens_ctx* c) {
    if (!c) return fail(nullptr, ENS_E_ARG, "ctx is NULL");
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    unsigned long long flag = 0;
    CUDA_TRY(c, cudaMemcpy(&flag, c->d_flag, sizeof(flag), cudaMemcpyDeviceToHost));
    if (flag != ~0ull) {
        c->latched = true;
        return fail(c, ENS_E_DIVERGED, "non-finite displacement at step " + std::to_string(flag >> 24) +
                                           " in realisation " + std::to_string(flag & 0xffffff));
    }
    return ENS_OK;
}

int ens_get_state(ens_ctx* c, double* u_n, double* u_nm1, double* t, int64_t* step) {
    if (!c) return fail(nullptr, ENS_E_ARG, "ctx is NULL");
    int rc = ens_sync(c);
    const size_t n = size_t(c->V) * 3 * size_t(c->n_s);
    double* cur = (c->step & 1) ? c->d_u1 : c->d_u0;
    double* old = (c->step & 1) ? c->d_u0 : c->d_u1;
    double* outs[2] = {u_n, u_nm1};
    double* srcs[2] = {cur, old};
    for (int k = 0; k < 2; ++k) {
        if (!outs[k]) continue;
        CUDA_TRY(c, ens::launch_dev_to_abi(c->V, c->n_s, c->d_perm, srcs[k], c->d_stage, c->stream));
        CUDA_TRY(c, cudaMemcpyAsync(outs[k], c->d_stage, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    }
    if (t) *t = double(c->step) * c->dt;
    if (step) *step = c->step;
    return rc;
}

int ens_set_state(ens_ctx* c, const double* u_n, const double* u_nm1, double t, int64_t step) {
    if (!c) return fail(nullptr, ENS_E_ARG, "ctx is NULL");
    if (step < 0) return fail(c, ENS_E_ARG, "step must be >= 0");
    (void)t;   // t = step * dt by construction
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    const size_t n = size_t(c->V) * 3 * size_t(c->n_s);
    double* cur = (step & 1) ? c->d_u1 : c->d_u0;
    double* old = (step & 1) ? c->d_u0 : c->d_u1;
    const double* ins[2] = {u_n, u_nm1};
    double* dsts[2] = {cur, old};
    for (int k = 0; k < 2; ++k) {
        if (!ins[k]) {
            CUDA_TRY(c, cudaMemsetAsync(dsts[k], 0, n * sizeof(double), c->stream));
            continue;
        }
        CUDA_TRY(c, cudaMemcpyAsync(c->d_stage, ins[k], n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(c, ens::launch_abi_to_dev(c->V, c->n_s, c->d_perm, c->d_stage, dsts[k], c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    }
    static thread_local int64_t h_step;
    h_step = step;
    CUDA_TRY(c, cudaMemcpyAsync(c->d_step, &h_step, sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaMemsetAsync(c->d_flag, 0xff, sizeof(unsigned long long), c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    c->step = step;
    c->latched = false;
    return ENS_OK;
}

int ens_apply_stiffness(ens_ctx* c, const double* u, double* y) {
    if (!c || !u || !y) return fail(c, ENS_E_ARG, "ens_apply_stiffness: NULL argument");
    const size_t n = size_t(c->V) * 3 * size_t(c->n_s);
    int rc;
    if (!c->d_scratch_u && ((rc = dalloc(c, &c->d_scratch_u, n)) || (rc = dalloc(c, &c->d_scratch_y, n)))) return rc;
    CUDA_TRY(c, cudaMemcpyAsync(c->d_stage, u, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, ens::launch_abi_to_dev(c->V, c->n_s, c->d_perm, c->d_stage, c->d_scratch_u, c->stream));
    ens::StepArgs a = step_args(c);
    a.ubuf0 = a.ubuf1 = c->d_scratch_u;
    a.y_out = c->d_scratch_y;
    CUDA_TRY(c, launch(c, a));
    CUDA_TRY(c, ens::launch_dev_to_abi(c->V, c->n_s, c->d_perm, c->d_scratch_y, c->d_stage, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(y, c->d_stage, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return ENS_OK;
}

int ens_query(const ens_ctx* c, ens_info* info) {
    if (!c || !info) return fail(nullptr, ENS_E_ARG, "NULL argument");
    std::memset(info, 0, sizeof(*info));
    info->dt = c->dt;
    info->dt_cfl = c->dt_cfl;
    info->n_nodes = c->V;
    info->n_tris = c->F;
    info->nnzb = c->nnzb;
    info->n_s = c->n_s;
    info->kernel = c->kernel;
    info->damping = c->damping;
    info->dist = c->dist;
    info->step = c->step;
    info->device_bytes = c->device_bytes;
    info->rcm_bandwidth = c->bandwidth;
    info->launches_per_step = 1;
    info->graph_steps = c->graph_steps;
    // algorithmic bytes: values + state read/read/write + c1 (+ c2, c3)
    const int64_t ns = c->n_s, per_node_state = 3 * 8 * 3 + 8 + (c->d_c2a ? 16 : 0);
    if (c->kernel == ENS_KERNEL_ASSEMBLED) {
        info->bytes_per_step = ns * (72 * c->nnzb + per_node_state * c->V);
        info->flops_per_step = ns * (18 * c->nnzb + 3 * 5 * c->V);
    } else {
        info->bytes_per_step = ns * (8 * c->F + per_node_state * c->V) + 648 * c->F;
        info->flops_per_step = ns * (3 * c->F * 60 + 3 * 5 * c->V);
    }
    return ENS_OK;
}

void ens_destroy(ens_ctx* c) {
    if (!c) return;
    if (c->stream) cudaStreamSynchronize(c->stream);
    drop_graph(c);
    free_all(c);
    delete c;
}

const char* ens_last_error(const ens_ctx* c) { return c ? c->err.c_str() : g_err.c_str(); }

// ---- host-side maps ------------------------------------------------------------------

int ens_host_validate(int64_t n_nodes, int64_t n_tris, const double* xyz, const int32_t* tris, int32_t* code,
                      int64_t* bad) {
    ens::MeshView m{n_nodes, n_tris, xyz, tris};
    int64_t b = -1;
    int v = ens::validate_mesh(m, &b);
    if (code) *code = v;
    if (bad) *bad = b;
    return v ? ENS_E_MESH : ENS_OK;
}

int ens_host_pattern(int64_t n_nodes, int64_t n_tris, const int32_t* tris, int32_t* perm, int64_t* row_ptr,
                     int32_t* col, int64_t col_cap, int64_t* nnzb) {
    ens::MeshView m{n_nodes, n_tris, nullptr, tris};
    ens::Pattern p = ens::build_pattern(m);
    *nnzb = int64_t(p.col.size());
    if (*nnzb > col_cap) return fail(nullptr, ENS_E_ARG, "col_cap too small");
    std::copy(p.perm.begin(), p.perm.end(), perm);
    std::copy(p.row_ptr.begin(), p.row_ptr.end(), row_ptr);
    std::copy(p.col.begin(), p.col.end(), col);
    return ENS_OK;
}

int ens_host_partition(int64_t n_nodes, const int64_t* row_ptr, int32_t n_parts, int64_t* bounds) {
    if (n_parts < 1) return fail(nullptr, ENS_E_ARG, "n_parts must be >= 1");
    std::vector<int64_t> rp(row_ptr, row_ptr + n_nodes + 1);
    auto b = ens::partition_bounds(rp, n_parts);
    std::copy(b.begin(), b.end(), bounds);
    return ENS_OK;
}

int ens_host_ghosts(int64_t n_nodes, const int64_t* row_ptr, const int32_t* col, int64_t lo, int64_t hi,
                    int32_t* ghosts, int64_t cap, int64_t* n) {
    std::vector<int64_t> rp(row_ptr, row_ptr + n_nodes + 1);
    std::vector<int32_t> cl(col, col + row_ptr[n_nodes]);
    auto g = ens::ghost_rows(rp, cl, lo, hi);
    *n = int64_t(g.size());
    if (*n > cap) return fail(nullptr, ENS_E_ARG, "cap too small");
    std::copy(g.begin(), g.end(), ghosts);
    return ENS_OK;
}

int ens_host_element_stiffness(int64_t n_nodes, int64_t n_tris, const double* xyz, const int32_t* tris, double nu,
                               double k_shear, double* Khat, double* area) {
    (void)n_nodes;
    for (int64_t e = 0; e < n_tris; ++e)
        ens::element_stiffness(xyz + 3 * int64_t(tris[3 * e]), xyz + 3 * int64_t(tris[3 * e + 1]),
                               xyz + 3 * int64_t(tris[3 * e + 2]), nu, k_shear, Khat + 81 * e, area + e);
    return ENS_OK;
}

int ens_host_materials(int64_t n_nodes, int64_t n_tris, const double* xyz, const int32_t* tris, int32_t n_s,
                       const double* E, const double* h, double rho, double cfl_safety, double* alpha, double* mass,
                       double* dt_cfl) {
    ens::MeshView m{n_nodes, n_tris, xyz, tris};
    ens::materials(m, n_s, E, h, rho, alpha, mass);
    if (dt_cfl) *dt_cfl = ens::cfl_dt(m, n_s, E, rho, cfl_safety > 0 ? cfl_safety : 0.9);
    return ENS_OK;
}

}  // extern "C"
