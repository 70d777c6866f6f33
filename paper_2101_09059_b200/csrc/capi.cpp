// capi.cpp -- the C ABI of include/ens.h: context lifetime, host setup -> device upload,
// step enqueue (fused kernels + halo exchange), state transfer.  Every step of the hot
// path runs in kernels.cu; the halo moves with NCCL (one part per process) or device
// copies (all parts in one context: the single-process emulation used by the tests).
#include "ens.h"

#include <algorithm>
#include <iterator>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "device.hpp"
#include "host_setup.hpp"
#include "nccl_dl.hpp"
#include "gmrf.hpp"
#include "observe.hpp"
#include "reassemble.hpp"

namespace {

thread_local std::string g_err;

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
};

// Matrix-free F3 tiles of one launched row range [row0, row0 + rows) (device.hpp MfTile).
struct MfTileSet {
    int64_t row0 = 0, rows = 0;
    int32_t ntiles = 0, stage_bytes = 0;
    ens::MfTile* d_tiles = nullptr;
    int4* d_entries = nullptr;
    unsigned char* d_blob = nullptr;
};

// One node partition held on this device: owned rows [lo, hi) of the RCM order, ghosts.
struct Part {
    ens::PartPlan plan;
    int64_t n_own = 0, n_gh = 0;
    int32_t *d_row_ptr = nullptr, *d_col = nullptr;
    int32_t *d_map_own = nullptr, *d_map_all = nullptr;   // local row -> caller node id
    int32_t* d_map_abi = nullptr;                          // owned row -> row of the ABI arrays
    int32_t* d_send_rows = nullptr;
    double *d_Kval = nullptr, *d_c1 = nullptr, *d_c2a = nullptr, *d_c3a = nullptr, *d_Fk = nullptr;
    double *d_u0 = nullptr, *d_u1 = nullptr, *d_sendbuf = nullptr;
    uint8_t* d_fixed = nullptr;
    int32_t* d_inc_ptr = nullptr;
    int4* d_fan = nullptr;
    int32_t* d_item_ptr = nullptr;                         // matrix-free item programs (F2w)
    int4* d_items = nullptr;
    double *d_Krow = nullptr, *d_alpha = nullptr;
    int32_t mf_rows = 1, mf_groups = 1, mf_smem_inc = 0;
    std::vector<MfTileSet> mfs;                            // matrix-free F3 tiles, per launched row range
    int64_t n_alpha = 0;                                   // alpha rows (elements touching the owned rows)
    int32_t *d_sym_lptr = nullptr, *d_sym_lidx = nullptr, *d_sym_lcol = nullptr, *d_sym_scol = nullptr;
    int2* d_sym_urange = nullptr;
    int64_t n_stored = 0;                                  // value blocks held (assembled kernels)
    // geometry-updated re-assembly (reassemble_every > 0): F0 inputs kept on the device
    int32_t *d_rcp = nullptr, *d_rcc = nullptr, *d_retri = nullptr;
    double *d_ral = nullptr, *d_rxyz = nullptr;
    double *d_scratch_u = nullptr, *d_scratch_y = nullptr;
    std::vector<int32_t> map_own;                          // host copy (ens_get_owned)
    // P2P halo (ENS_HALO_P2P): forward lists, neighbour tables, own flags
    unsigned long long* d_hflags = nullptr;                // [world]: step published by neighbour q
    int32_t* d_fwd_ptr = nullptr;                          // [n_own + 1]
    int2* d_fwd_dst = nullptr;                             // {slot, peer local row}
    double** d_peer_buf = nullptr;                         // [2 n_out]
    unsigned long long** d_out_flag = nullptr;             // [n_out]: &flags_q[p] of neighbour q
    int32_t* d_in_q = nullptr;                             // [n_in] neighbours this part waits for
    unsigned int* d_hdone = nullptr;                       // CTAs done in the publishing launch (hw_signal)
    int32_t n_out = 0, n_in = 0;
    std::vector<int32_t> out_q;                            // neighbour rank of each slot
    std::vector<int64_t> out_rows;                         // its local row count (owned + ghosts)
};

}  // namespace

struct ens_ctx {
    std::string err;
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t comm_stream = nullptr;
    cudaEvent_t ev_packed = nullptr, ev_halo = nullptr;
    void* (*dev_alloc)(size_t, void*) = nullptr;
    void (*dev_free)(void*, void*) = nullptr;
    void* alloc_user = nullptr;
    std::vector<DevBuf> bufs;
    int64_t device_bytes = 0;

    int64_t V = 0, F = 0, nnzb = 0;
    int32_t n_s = 0, s_begin = 0;
    int32_t kernel = 0, damping = 0, dist = 0, rank = 0, world = 1;
    int32_t mf_variant = 0;                 // matrix-free data path in use (ENS_MF_*), resolved at create
    ens::MfsPlan mfs_plan;                  // F3 shape and tiling (kernels.cu mf_staged_plan)
    double dt = 0.0, dt_cfl = 0.0, c_d = 0.0;
    double c2 = 2.0, c3 = 1.0;
    int32_t bandwidth = 0;
    std::vector<int32_t> perm, iperm;       // perm[new] = old (global)

    std::vector<Part> parts;                // 1 (single / ensemble / one rank) or world (emulation)
    const ens::Nccl* nccl = nullptr;
    void* nccl_comm = nullptr;
    int32_t halo = ENS_HALO_NCCL;
    bool multi = false;                     // this process holds one part of `world` (NCCL or IPC)
    bool p2p_connected = true;              // IPC peers opened (ens_p2p_connect)
    unsigned long long* d_herr = nullptr;   // P2P wait timeout: step << 16 | neighbour
    std::vector<void*> raw_bufs;            // cudaMalloc'd (IPC-exported) buffers
    std::vector<void*> ipc_opened;          // neighbours' buffers opened by ens_p2p_connect

    double* d_stage = nullptr;              // [n_s][V][3] ABI staging
    unsigned long long* d_flag = nullptr;
    double* d_coef = nullptr;               // [2][kMaxFields] load coefficients (StepArgs.coef_buf)
    // asynchronous traction updates (same shape): host staging in pinned memory
    double* h_trac = nullptr;
    size_t h_trac_n = 0;
    cudaEvent_t ev_trac = nullptr;          // the last traction H2D copy has consumed h_trac
    // asynchronous observation (ens_observe): transpose on the stream, D2H on obs_stream
    cudaStream_t obs_stream = nullptr;
    cudaEvent_t ev_obs_ready = nullptr, ev_obs_done = nullptr;
    double* d_obs = nullptr;
    unsigned long long* h_obs_flag = nullptr;   // pinned copy of d_flag taken with the snapshot
    bool obs_pending = false;
    int64_t obs_step = 0;
    bool coef_dirty = true;                 // seed d_coef before the next step
    int64_t* d_step = nullptr;
    int32_t n_fields = 0, n_tab = 0;
    double *d_tab_t = nullptr, *d_tab_g = nullptr;
    double period = 0.0, ramp_T = 0.0;

    int64_t step = 0;
    bool latched = false;
    int32_t reassemble_every = 0;

    // observation (stresses, statistics): host mesh copy, element E means, lazy operators
    std::vector<double> h_xyz;
    std::vector<int32_t> h_tris;
    double nu = 0.0, k_shear = 0.0;
    double* d_Ebar = nullptr;               // [F][n_s]
    double* d_G = nullptr;                  // [F][45]
    int32_t* d_etri = nullptr;              // [F][3] RCM ids

    bool persistent = false;                // N2: one persistent kernel per ens_step (ens_options.persistent)
    ens::StepArgs* d_pparts = nullptr;      // its per-part arguments (rebuilt when the graphs would be)
    int64_t* d_pitems = nullptr;            // [parts + 1] prefix of (row, group) items
    unsigned int* d_pbar = nullptr;         // grid-barrier state [2]
    int32_t graph_steps = 64;               // CUDA graph of this many steps (single part, no halo)
    // one graph per parity of the step it starts at: the NCCL / device-copy halos receive
    // into buffer (step + 1) & 1, fixed in the captured nodes (the kernels read the step
    // from the device counter and need no such split)
    cudaGraphExec_t graph[2] = {nullptr, nullptr};
    bool graph_dirty = true;

    bool has_halo() const { return parts.size() > 1 || multi; }
    bool p2p() const { return has_halo() && halo == ENS_HALO_P2P; }
    // the step loop runs as CUDA graphs of graph_steps steps with every halo: the NCCL
    // send/recv (captured on the comm stream forked from the step stream), the device-copy
    // emulation and the P2P flags are all capturable; re-assembly steps are not
    bool use_graphs() const { return graph_steps > 0 && reassemble_every == 0; }
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

#define CUDA_TRY(c, expr)                                      \
    do {                                                       \
        cudaError_t _e = (expr);                               \
        if (_e != cudaSuccess) return cuda_fail(c, _e, #expr); \
    } while (0)

#define RC_TRY(expr)              \
    do {                          \
        int _rc = (expr);         \
        if (_rc) return _rc;      \
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
int rawalloc(ens_ctx* c, T** out, size_t count) {
    *out = nullptr;
    const size_t bytes = std::max<size_t>(count * sizeof(T), 16);
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) return cuda_fail(c, e, "cudaMalloc (IPC-exported buffer)");
    c->raw_bufs.push_back(p);
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
    RC_TRY(dalloc(c, out, count));
    if (count) CUDA_TRY(c, cudaMemcpyAsync(*out, host, count * sizeof(T), cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));   // host staging vectors are temporaries
    return ENS_OK;
}

void drop_graph(ens_ctx* c) {
    for (auto& g : c->graph) {
        if (g) cudaGraphExecDestroy(g);
        g = nullptr;
    }
    c->graph_dirty = true;
}

void free_all(ens_ctx* c) {
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->obs_stream) cudaStreamSynchronize(c->obs_stream);
    drop_graph(c);
    if (c->h_trac) cudaFreeHost(c->h_trac);
    if (c->h_obs_flag) cudaFreeHost(c->h_obs_flag);
    if (c->ev_trac) cudaEventDestroy(c->ev_trac);
    if (c->obs_stream) cudaStreamDestroy(c->obs_stream);
    if (c->ev_obs_ready) cudaEventDestroy(c->ev_obs_ready);
    if (c->ev_obs_done) cudaEventDestroy(c->ev_obs_done);
    c->h_trac = nullptr;
    c->h_obs_flag = nullptr;
    c->ev_trac = c->ev_obs_ready = c->ev_obs_done = nullptr;
    c->obs_stream = nullptr;
    for (void* p : c->ipc_opened) cudaIpcCloseMemHandle(p);
    c->ipc_opened.clear();
    for (void* p : c->raw_bufs) cudaFree(p);
    c->raw_bufs.clear();
    for (auto& b : c->bufs) {
        if (c->dev_free) c->dev_free(b.p, c->alloc_user);
        else cudaFreeAsync(b.p, c->stream);
    }
    if (c->stream) cudaStreamSynchronize(c->stream);
    c->bufs.clear();
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    if (c->ev_packed) cudaEventDestroy(c->ev_packed);
    if (c->ev_halo) cudaEventDestroy(c->ev_halo);
    c->comm_stream = nullptr;
    c->ev_packed = c->ev_halo = nullptr;
}

int check_opts(const ens_options* opt) {
    if (!opt) return ENS_OK;
    if (!(std::isfinite(opt->dt))) return fail(nullptr, ENS_E_ARG, "opt->dt is not finite");
    if (opt->damping < 0 || opt->damping > 2) return fail(nullptr, ENS_E_ARG, "opt->damping must be 0, 1 or 2");
    if (opt->kernel < 0 || opt->kernel > 2) return fail(nullptr, ENS_E_ARG, "opt->kernel must be 0, 1 or 2");
    if (!(opt->c_d >= 0.0) || !std::isfinite(opt->c_d)) return fail(nullptr, ENS_E_ARG, "opt->c_d must be finite and >= 0");
    if (opt->dist < 0 || opt->dist > 2) return fail(nullptr, ENS_E_ARG, "opt->dist must be 0, 1 or 2");
    if (opt->reassemble_every < 0) return fail(nullptr, ENS_E_ARG, "opt->reassemble_every must be >= 0");
    if (opt->reassemble_every > 0 && opt->kernel == ENS_KERNEL_MATRIX_FREE)
        return fail(nullptr, ENS_E_UNSUPPORTED,
                    "reassemble_every needs an assembled kernel (per-realisation geometry breaks the shared K^_e)");
    if (opt->halo < 0 || opt->halo > 1) return fail(nullptr, ENS_E_ARG, "opt->halo must be 0 (NCCL) or 1 (P2P)");
    if (opt->mf_variant < 0 || opt->mf_variant > 3) return fail(nullptr, ENS_E_ARG, "opt->mf_variant must be 0..3 (ENS_MF_*)");
    if (opt->persistent && (opt->dist != ENS_DIST_NODE || opt->halo != ENS_HALO_P2P ||
                            opt->kernel == ENS_KERNEL_MATRIX_FREE || opt->reassemble_every > 0))
        return fail(nullptr, ENS_E_UNSUPPORTED,
                    "opt->persistent needs dist = NODE, halo = P2P, an assembled kernel and no re-assembly");
    if (opt->p2p_procs && (opt->halo != ENS_HALO_P2P || opt->dist != ENS_DIST_NODE))
        return fail(nullptr, ENS_E_ARG, "opt->p2p_procs needs dist = NODE and halo = P2P");
    if (opt->halo == ENS_HALO_P2P && opt->nccl_comm)
        return fail(nullptr, ENS_E_ARG, "opt->halo = P2P takes no nccl_comm");
    if (opt->dist == ENS_DIST_NODE) {
        if (opt->world < 1) return fail(nullptr, ENS_E_ARG, "opt->world must be >= 1");
        if ((opt->nccl_comm || opt->p2p_procs) && (opt->rank < 0 || opt->rank >= opt->world))
            return fail(nullptr, ENS_E_ARG, "opt->rank must lie in [0, world)");
    }
    return ENS_OK;
}

int init_ctx(ens_ctx* c, const ens_options* opt) {
    ens_options def{};
    def.device = -1;
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
    c->rank = opt->rank;
    c->world = opt->world > 0 ? opt->world : 1;
    c->reassemble_every = opt->reassemble_every;
    c->persistent = opt->persistent != 0;
    c->nccl_comm = opt->dist == ENS_DIST_NODE ? opt->nccl_comm : nullptr;
    c->halo = opt->dist == ENS_DIST_NODE ? opt->halo : ENS_HALO_NCCL;
    c->multi = c->nccl_comm != nullptr || (c->halo == ENS_HALO_P2P && opt->p2p_procs != 0 && c->world > 1);
    c->p2p_connected = !(c->multi && c->halo == ENS_HALO_P2P);
    if (c->nccl_comm) {
        std::string why;
        c->nccl = ens::nccl_load(&why);
        if (!c->nccl) return fail(c, ENS_E_NCCL, why);
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_packed, cudaEventDisableTiming));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
    }
    if (const char* g = std::getenv("ENS_GRAPH_STEPS")) c->graph_steps = std::max(0, std::atoi(g));
    return ENS_OK;
}

ens::StepArgs part_args(const ens_ctx* c, const Part& p) {
    ens::StepArgs a;
    a.row0 = 0;
    a.V = p.n_own;
    a.fk_rows = p.n_own;
    a.n_s = c->n_s;
    a.row_ptr = p.d_row_ptr;
    a.col = p.d_col;
    a.Kval = p.d_Kval;
    a.inc_ptr = p.d_inc_ptr;
    a.fan = p.d_fan;
    a.item_ptr = p.d_item_ptr;
    a.items = p.d_items;
    a.Krow = p.d_Krow;
    a.alpha = p.d_alpha;
    a.mf_rows = p.mf_rows;
    a.mf_groups = p.mf_groups;
    a.mf_smem_inc = p.mf_smem_inc;
    a.sym_lptr = p.d_sym_lptr;
    a.sym_lidx = p.d_sym_lidx;
    a.sym_lcol = p.d_sym_lcol;
    a.sym_urange = p.d_sym_urange;
    a.sym_scol = p.d_sym_scol;
    a.c1 = p.d_c1;
    a.c2a = p.d_c2a;
    a.c3a = p.d_c3a;
    a.c2 = c->c2;
    a.c3 = c->c3;
    a.fixed = p.d_fixed;
    a.n_fields = c->n_fields;
    a.Fk = p.d_Fk;
    a.n_tab = c->n_tab;
    a.tab_t = c->d_tab_t;
    a.tab_g = c->d_tab_g;
    a.period = c->period;
    a.ramp_T = c->ramp_T;
    a.dt = c->dt;
    a.step_base = c->d_step;
    a.ubuf0 = p.d_u0;
    a.ubuf1 = p.d_u1;
    a.u_rows = p.n_own + p.n_gh;
    a.flag = c->d_flag;
    a.coef_buf = c->d_coef;
    a.s_global0 = c->s_begin;
    return a;
}

cudaError_t launch_rows(const ens_ctx* c, const Part& p, ens::StepArgs a, int64_t row0, int64_t rows, cudaStream_t st) {
    if (rows <= 0) return cudaSuccess;
    a.row0 = row0;
    a.V = rows;
    if (c->kernel == ENS_KERNEL_MATRIX_FREE && c->mf_variant == ENS_MF_STAGED) {
        // the tile set built for exactly this row range (build_part)
        const MfTileSet* ts = nullptr;
        for (const MfTileSet& t : p.mfs)
            if (t.row0 == row0 && t.rows == rows) ts = &t;
        if (!ts) return cudaErrorInvalidValue;
        a.mfs_tiles = ts->d_tiles;
        a.mfs_entries = ts->d_entries;
        a.mfs_blob = ts->d_blob;
        a.mfs_ntiles = ts->ntiles;
        a.mfs_stage_bytes = ts->stage_bytes;
        a.mfs_shape = c->mfs_plan.shape;
        a.mfs_slices = c->mfs_plan.sliced ? (c->n_s + ens::mfs_stage_w(c->mfs_plan, c->n_s) - 1) /
                                                 ens::mfs_stage_w(c->mfs_plan, c->n_s) : 1;
        a.mfs_alpha_rows = p.n_alpha;
    }
    switch (c->kernel) {
        case ENS_KERNEL_MATRIX_FREE: return ens::launch_step_matrix_free(a, st);
        case ENS_KERNEL_ASSEMBLED_SYM: return ens::launch_step_assembled_sym(a, st);
        default: return ens::launch_step_assembled(a, st);
    }
}

// ---- one time step of every part (step index = ctx step + k) ---------------------------
int reassemble_if_due(ens_ctx* c, Part& p, int64_t step, cudaStream_t st) {
    if (c->reassemble_every > 0 && step > 0 && step % c->reassemble_every == 0)   // K_s(X + u_step)
        CUDA_TRY(c, ens::launch_reassemble(p.n_stored, c->n_s, p.d_rcp, p.d_rcc, p.d_ral, p.d_retri, p.d_rxyz,
                                           (step & 1) ? p.d_u1 : p.d_u0, c->nu, c->k_shear, p.d_Kval, st));
    return ENS_OK;
}

// Steps with a halo run on two streams: the halo chain (boundary rows of every part, which
// read ghosts and which the neighbours need, then the exchange) on comm_stream, the
// interior rows (no ghost column) on the step stream; both join before the next step,
// since each half reads the other's u_{n+1} next step.  A step that re-assembles first
// runs serially on the step stream.
bool reassembly_due(const ens_ctx* c, int64_t step) {
    return c->reassemble_every > 0 && step > 0 && step % c->reassemble_every == 0;
}

int fork_halo(ens_ctx* c, cudaStream_t st, bool fork, cudaStream_t* hs) {
    *hs = fork ? c->comm_stream : st;
    if (fork) {
        CUDA_TRY(c, cudaEventRecord(c->ev_packed, st));
        CUDA_TRY(c, cudaStreamWaitEvent(c->comm_stream, c->ev_packed, 0));
    }
    return ENS_OK;
}

int join_halo(ens_ctx* c, cudaStream_t st, bool fork) {
    if (fork) {
        CUDA_TRY(c, cudaEventRecord(c->ev_halo, c->comm_stream));
        CUDA_TRY(c, cudaStreamWaitEvent(st, c->ev_halo, 0));
    }
    return ENS_OK;
}

int launch_interior(ens_ctx* c, int64_t k, cudaStream_t st) {
    for (Part& p : c->parts) {
        ens::StepArgs a = part_args(c, p);
        a.step_off = k;
        CUDA_TRY(c, launch_rows(c, p, a, p.plan.b_lo, p.n_own - p.plan.b_lo - p.plan.b_hi, st));
    }
    return ENS_OK;
}

// P2P halo step (ENS_HALO_P2P): per part, wait for the neighbours' u_n ghost
// rows (their flags >= step), boundary rows with u_{n+1} forwarded into the neighbours'
// ghost rows of buffer (step + 1) & 1, publish step + 1 — all on the halo stream, while
// the interior rows run on the step stream.  Neighbours only ever write ghost rows of the
// buffer this part is not reading, and only after it published the step before, so two
// buffers suffice (no acknowledgement needed).
// The step kernels a1, a1s and F3 wait for the neighbours' flags and publish their own inside
// the boundary-row launches (StepArgs::hw_*): 3 launches per part per step instead of 5
// (ENS_HALO_FUSED=0 restores the separate k_halo_wait / k_halo_signal launches).
bool halo_fused(const ens_ctx* c) {
    static const bool on = [] {
        const char* e = std::getenv("ENS_HALO_FUSED");
        return e ? std::atoi(e) != 0 : true;
    }();
    return on && (c->kernel != ENS_KERNEL_MATRIX_FREE || c->mf_variant == ENS_MF_STAGED);
}

int enqueue_step_p2p(ens_ctx* c, int64_t step0, int64_t k, cudaStream_t st) {
    const int64_t step = step0 + k;
    const bool fork = !reassembly_due(c, step);
    cudaStream_t hs;
    RC_TRY(fork_halo(c, st, fork, &hs));
    for (Part& p : c->parts) {
        ens::StepArgs a = part_args(c, p);
        a.step_off = k;
        a.fwd_ptr = p.d_fwd_ptr;
        a.fwd_dst = p.d_fwd_dst;
        a.peer_buf = p.d_peer_buf;
        const bool fused = halo_fused(c) && fork && (p.plan.b_lo > 0 || p.plan.b_hi > 0);
        if (!fused) {
            CUDA_TRY(c, ens::launch_halo_wait(p.n_in, p.d_in_q, p.d_hflags, c->d_step, k, c->d_herr, hs));
            RC_TRY(reassemble_if_due(c, p, step, hs));
            CUDA_TRY(c, launch_rows(c, p, a, 0, p.plan.b_lo, hs));
            CUDA_TRY(c, launch_rows(c, p, a, p.n_own - p.plan.b_hi, p.plan.b_hi, hs));
            CUDA_TRY(c, ens::launch_halo_signal(p.n_out, p.d_out_flag, c->d_step, k, hs));
            continue;
        }
        // the first boundary launch waits, the last one publishes
        ens::StepArgs w = a, g = a;
        w.hw_wait = p.n_in > 0;
        w.hw_flags = p.d_hflags;
        w.hw_in_q = p.d_in_q;
        w.hw_n_in = p.n_in;
        w.hw_err = c->d_herr;
        g.hw_signal = p.n_out > 0;
        g.hw_out = p.d_out_flag;
        g.hw_n_out = p.n_out;
        g.hw_done = p.d_hdone;
        if (p.plan.b_lo > 0 && p.plan.b_hi > 0) {
            CUDA_TRY(c, launch_rows(c, p, w, 0, p.plan.b_lo, hs));
            CUDA_TRY(c, launch_rows(c, p, g, p.n_own - p.plan.b_hi, p.plan.b_hi, hs));
        } else {
            ens::StepArgs b = w;
            b.hw_signal = g.hw_signal;
            b.hw_out = g.hw_out;
            b.hw_n_out = g.hw_n_out;
            b.hw_done = g.hw_done;
            if (p.plan.b_lo > 0) CUDA_TRY(c, launch_rows(c, p, b, 0, p.plan.b_lo, hs));
            else CUDA_TRY(c, launch_rows(c, p, b, p.n_own - p.plan.b_hi, p.plan.b_hi, hs));
        }
    }
    RC_TRY(launch_interior(c, k, st));
    return join_halo(c, st, fork);
}

// step0: the host mirror of *d_step when the step runs (c->step for direct launches; a step
// of the right parity when captured into a graph)
int enqueue_step(ens_ctx* c, int64_t step0, int64_t k, cudaStream_t st) {
    const int64_t step = step0 + k;              // host mirror of *d_step + k
    if (c->p2p()) return enqueue_step_p2p(c, step0, k, st);
    for (Part& p : c->parts) RC_TRY(reassemble_if_due(c, p, step, st));
    if (!c->has_halo()) {
        ens::StepArgs a = part_args(c, c->parts[0]);
        a.step_off = k;
        CUDA_TRY(c, launch_rows(c, c->parts[0], a, 0, c->parts[0].n_own, st));
        return ENS_OK;
    }
    cudaStream_t hs;
    RC_TRY(fork_halo(c, st, true, &hs));
    // (1) boundary rows of every part (they read ghosts, and the neighbours need them)
    for (Part& p : c->parts) {
        ens::StepArgs a = part_args(c, p);
        a.step_off = k;
        CUDA_TRY(c, launch_rows(c, p, a, 0, p.plan.b_lo, hs));
        CUDA_TRY(c, launch_rows(c, p, a, p.n_own - p.plan.b_hi, p.plan.b_hi, hs));
        CUDA_TRY(c, ens::launch_pack(int64_t(p.plan.send_rows.size()), c->n_s, p.d_send_rows, c->d_step, k, p.d_u0,
                                     p.d_u1, p.d_sendbuf, hs));
    }
    const size_t w = size_t(3) * size_t(c->n_s);
    auto unew = [&](Part& p) { return ((step + 1) & 1) ? p.d_u1 : p.d_u0; };
    // (2) halo: u_{n+1} of the send rows -> the neighbours' ghost rows
    if (c->nccl_comm) {
        Part& p = c->parts[0];
        const ens::Nccl& N = *c->nccl;
        int r = N.group_start();
        for (const auto& pe : p.plan.peers) {
            if (r == 0 && pe.send_n)
                r = N.send(p.d_sendbuf + size_t(pe.send_off) * w, size_t(pe.send_n) * w, ens::Nccl::kDouble, pe.q,
                           c->nccl_comm, hs);
            if (r == 0 && pe.recv_n)
                r = N.recv(unew(p) + size_t(pe.recv_row) * w, size_t(pe.recv_n) * w, ens::Nccl::kDouble, pe.q,
                           c->nccl_comm, hs);
        }
        int r2 = N.group_end();
        if (r == 0) r = r2;
        if (r != 0)
            return fail(c, ENS_E_NCCL, std::string("halo exchange: ") + (N.error_string ? N.error_string(r) : "error"));
    } else {
        for (Part& p : c->parts)
            for (const auto& pe : p.plan.peers) {
                if (!pe.recv_n) continue;
                const Part& q = c->parts[size_t(pe.q)];
                const auto it = std::find_if(q.plan.peers.begin(), q.plan.peers.end(),
                                             [&](const ens::PartPlan::Peer& x) { return x.q == p.plan.p; });
                CUDA_TRY(c, cudaMemcpyAsync(unew(p) + size_t(pe.recv_row) * w, q.d_sendbuf + size_t(it->send_off) * w,
                                            size_t(pe.recv_n) * w * sizeof(double), cudaMemcpyDeviceToDevice, hs));
            }
    }
    // (3) interior rows on the step stream, overlapping (1)-(2); (4) join
    RC_TRY(launch_interior(c, k, st));
    return join_halo(c, st, true);
}

// Capture graph_steps steps + the counter advance on a private stream (the caller's stream
// may be the legacy default stream, which cannot capture).
int build_graph(ens_ctx* c, int parity) {
    cudaGraphExec_t& ge = c->graph[parity];
    if (ge) cudaGraphExecDestroy(ge);
    ge = nullptr;
    cudaStream_t cap = nullptr;
    CUDA_TRY(c, cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
    cudaError_t err = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
    int rc = ENS_OK;
    for (int32_t k = 0; err == cudaSuccess && rc == ENS_OK && k < c->graph_steps; ++k)
        rc = enqueue_step(c, parity, k, cap);
    if (err == cudaSuccess && rc == ENS_OK) err = ens::launch_advance(c->d_step, c->graph_steps, cap);
    cudaGraph_t g = nullptr;
    cudaError_t e2 = cudaStreamEndCapture(cap, &g);
    if (err == cudaSuccess) err = e2;
    if (err == cudaSuccess && rc == ENS_OK) err = cudaGraphInstantiate(&ge, g, 0);
    if (g) cudaGraphDestroy(g);
    cudaStreamDestroy(cap);
    if (rc) return rc;
    if (err != cudaSuccess) return cuda_fail(c, err, "CUDA graph capture of the step loop");
    return ENS_OK;
}

// ---- per-part device operator ---------------------------------------------------------
struct Global {
    const ens::MeshView* m;
    const ens::Pattern* pat;
    const std::vector<double>* Khat;       // [F][81]
    const std::vector<double>* alpha;      // [n_s][F]
    const std::vector<double>* mass;       // [n_s][V] caller numbering
    const uint8_t* fixed;                  // caller numbering or null
    const ens::Fans* fans;                 // matrix-free only
    const std::vector<int32_t>* contrib_ptr;   // [nnzb + 1] (assembled only)
    const std::vector<int32_t>* contrib;       // e * 9 + a * 3 + b
};

// ---- matrix-free F3 tiles (device.hpp MfTile, kernels.cu k_step_mf_staged) ---------------
// A tile is a compact patch of at most kMfsMaxRows rows: its stage holds the u_n rows of the
// patch and of its 1-ring, so a round patch moves fewer neighbour rows per own row than a
// strip of consecutive RCM rows (measured on c2: 6.3 vs 9.0 KB per row at 76 KB stages).
struct MfLayout {
    std::vector<int32_t> rows;                 // own rows (ascending)
    std::vector<int2> uspan, espan;            // other nodes / elements as spans {first, count}
    int64_t n_unodes = 0, n_elems = 0;         // rows in the spans (gaps included)
    size_t blob_bytes = 0, bytes = 0;          // bytes: blob + u + alpha (F_k budgeted separately)
    int entries = 0;
};

// spans covering the sorted ids v, merging gaps of at most `gap` ids (one copy each)
static void spans_of(const std::vector<int32_t>& v, int gap, std::vector<int2>& out, int64_t& total) {
    out.clear();
    total = 0;
    for (int32_t x : v) {
        if (!out.empty() && x - (out.back().x + out.back().y) <= gap) out.back().y = x - out.back().x + 1;
        else out.push_back(make_int2(x, 1));
    }
    for (const int2& sp : out) total += sp.y;
}

static int count_runs(const std::vector<int32_t>& v) {
    int n = 0;
    for (size_t k = 0; k < v.size(); ++k)
        if (k == 0 || v[k] != v[k - 1] + 1) ++n;
    return n;
}

// gaps merged into one bulk copy (ENS_MFS_GAP_U / _A): fewer TMA copies for a few more bytes
static int mfs_gap(bool u) {
    static const int gu = [] { const char* e = std::getenv("ENS_MFS_GAP_U"); return e ? std::atoi(e) : 0; }();
    static const int ga = [] { const char* e = std::getenv("ENS_MFS_GAP_A"); return e ? std::atoi(e) : 0; }();
    return u ? gu : ga;
}

static void mf_layout(const std::vector<int32_t>& ip, const std::vector<ens::FanRec>& rec, std::vector<int32_t> rows,
                      size_t US, size_t AS, MfLayout& L) {
    std::sort(rows.begin(), rows.end());
    L.rows = rows;
    std::vector<int32_t> nodes, elems, other;
    size_t ninc = 0;
    for (int32_t r : rows)
        for (int32_t k = ip[size_t(r)]; k < ip[size_t(r) + 1]; ++k) {
            nodes.push_back(rec[size_t(k)].n_prev);
            nodes.push_back(rec[size_t(k)].n_next);
            elems.push_back(rec[size_t(k)].e);
            ++ninc;
        }
    std::sort(nodes.begin(), nodes.end());
    nodes.erase(std::unique(nodes.begin(), nodes.end()), nodes.end());
    std::set_difference(nodes.begin(), nodes.end(), rows.begin(), rows.end(), std::back_inserter(other));
    std::sort(elems.begin(), elems.end());
    elems.erase(std::unique(elems.begin(), elems.end()), elems.end());
    spans_of(other, mfs_gap(true), L.uspan, L.n_unodes);
    spans_of(elems, mfs_gap(false), L.espan, L.n_elems);
    L.blob_bytes = (size_t(ens::kMfsHdrBytes) + ninc * ens::kMfsRecBytes + (2 * rows.size() + 1) * 4 + 127) & ~size_t(127);
    L.bytes = L.blob_bytes + (rows.size() + size_t(L.n_unodes)) * US + size_t(L.n_elems) * AS;
    const int own_runs = count_runs(rows);
    L.entries = 2 * own_runs + int(L.uspan.size() + L.espan.size()) + 1;   // u + F_k per own run
}

// Greedy patches of rows [row0, row0 + rows): seed = the first unassigned row (RCM order); grow
// by the unassigned neighbour adding the fewest new nodes to the tile's node set (ties: lowest
// id) while the stage image fits.
static std::vector<std::vector<int32_t>> mf_patches(const std::vector<int32_t>& ip, const std::vector<ens::FanRec>& rec,
                                                    int64_t n_loc, int64_t row0, int64_t rows, size_t US, size_t AS,
                                                    size_t SB, const ens::MfsPlan& plan) {
    auto nbrs = [&](int32_t r, std::vector<int32_t>& v) {
        v.clear();
        for (int32_t k = ip[size_t(r)]; k < ip[size_t(r) + 1]; ++k) {
            v.push_back(rec[size_t(k)].n_prev);
            v.push_back(rec[size_t(k)].n_next);
        }
        std::sort(v.begin(), v.end());
        v.erase(std::unique(v.begin(), v.end()), v.end());
    };
    std::vector<std::vector<int32_t>> tiles;
    MfLayout L;
    if (!plan.patches) {                   // strips of consecutive rows
        for (int64_t r = row0; r < row0 + rows;) {
            std::vector<int32_t> tile = {int32_t(r)};
            while (int(tile.size()) < plan.max_rows && r + int64_t(tile.size()) < row0 + rows) {
                tile.push_back(int32_t(r + int64_t(tile.size())));
                mf_layout(ip, rec, tile, US, AS, L);
                if (L.bytes + size_t(ens::kMaxFields) * tile.size() * 32 > SB || L.entries > ens::kMfsMaxEntries - 8) {
                    tile.pop_back();
                    break;
                }
            }
            r += int64_t(tile.size());
            tiles.push_back(tile);
        }
        return tiles;
    }
    std::vector<std::vector<int32_t>> nb(static_cast<size_t>(rows));
    for (int64_t r = 0; r < rows; ++r) nbrs(int32_t(row0 + r), nb[size_t(r)]);
    auto in_range = [&](int32_t x) { return x >= row0 && x < row0 + rows; };
    std::vector<char> assigned(static_cast<size_t>(rows), 0);
    std::vector<int32_t> mark(static_cast<size_t>(n_loc), -1);
    for (int64_t seed = row0; seed < row0 + rows; ++seed) {
        if (assigned[size_t(seed - row0)]) continue;
        const int32_t tid = int32_t(tiles.size());
        std::vector<int32_t> tile = {int32_t(seed)};
        assigned[size_t(seed - row0)] = 1;
        mark[size_t(seed)] = tid;
        for (int32_t z : nb[size_t(seed - row0)]) mark[size_t(z)] = tid;
        while (int(tile.size()) < plan.max_rows) {
            int32_t best = -1, bc = 1 << 30;
            for (int32_t x : tile)
                for (int32_t y : nb[size_t(x - row0)]) {
                    if (!in_range(y) || assigned[size_t(y - row0)]) continue;
                    int32_t cost = mark[size_t(y)] != tid;
                    for (int32_t z : nb[size_t(y - row0)]) cost += mark[size_t(z)] != tid;
                    if (cost < bc || (cost == bc && y < best)) { bc = cost; best = y; }
                }
            if (best < 0) break;
            tile.push_back(best);
            mf_layout(ip, rec, tile, US, AS, L);
            if (L.bytes + size_t(ens::kMaxFields) * tile.size() * 32 > SB || L.entries > ens::kMfsMaxEntries - 8) {
                tile.pop_back();
                break;
            }
            assigned[size_t(best - row0)] = 1;
            mark[size_t(best)] = tid;
            for (int32_t z : nb[size_t(best - row0)]) mark[size_t(z)] = tid;
        }
        tiles.push_back(tile);
    }
    return tiles;
}

// Bytes of a stage a tile image may fill.  With a ragged N_s in whole-row stages the lanes of
// a row's last (partial) unit read up to 8 * pad bytes past the end of a node row (pad = the
// realisations that round N_s up to whole units; kernels.cu k_step_mf_staged): that much
// slack stays free at the end of every stage.
static size_t mfs_budget(const ens_ctx* c, const ens::MfsShape& sh) {
    const int64_t w = 64 * c->mfs_plan.ws;
    const int64_t pad = c->mfs_plan.sliced ? 0 : (c->n_s + w - 1) / w * w - c->n_s;
    return size_t(sh.stage_bytes) - size_t((8 * pad + 127) & ~int64_t(127));
}

// Upload the tile set of one launched row range: copy entries and blobs (final element ids).
int build_mf_tiles(ens_ctx* c, const std::vector<int32_t>& ip, const std::vector<ens::FanRec>& rec,
                   const std::vector<double>& k18, const std::vector<uint8_t>& fx,
                   std::vector<std::vector<int32_t>> patches, int64_t row0, int64_t rows, MfTileSet& out) {
    const ens::MfsShape sh = ens::mf_staged_shape(c->mfs_plan.shape);
    const size_t W = size_t(ens::mfs_stage_w(c->mfs_plan, c->n_s));   // realisations per stage row
    const size_t US = W * 24, AS = W * 8;
    std::vector<ens::MfTile> tiles;
    std::vector<int4> entries;
    std::vector<unsigned char> blob;
    MfLayout L;
    for (size_t pi = 0; pi < patches.size(); ++pi) {
        mf_layout(ip, rec, patches[pi], US, AS, L);
        if (L.entries > ens::kMfsMaxEntries ||
            L.bytes + size_t(ens::kMaxFields) * L.rows.size() * 32 > mfs_budget(c, sh)) {
            if (L.rows.size() == 1)
                return fail(c, ENS_E_UNSUPPORTED, "matrix-free staged: the operands of row " +
                                                      std::to_string(L.rows[0]) + " exceed one shared-memory stage");
            const size_t h = L.rows.size() / 2;       // split and retry (element ids changed)
            patches.insert(patches.begin() + int64_t(pi) + 1, std::vector<int32_t>(L.rows.begin() + int64_t(h), L.rows.end()));
            patches[pi].assign(L.rows.begin(), L.rows.begin() + int64_t(h));
            --pi;
            continue;
        }
        const int32_t nr = int32_t(L.rows.size());
        const int32_t u_base = int32_t(L.blob_bytes);
        const int32_t a_base = int32_t(L.blob_bytes + (L.rows.size() + size_t(L.n_unodes)) * US);
        const int32_t f_base = int32_t(L.bytes);
        ens::MfTile t{};
        t.entry0 = int32_t(entries.size());
        t.nrows = nr;
        t.stage_bytes = int32_t(L.bytes);
        auto add_runs = [&](const std::vector<int32_t>& v, int kind, int32_t base, size_t unit) {
            for (size_t k = 0; k < v.size();) {
                size_t n = 1;
                while (k + n < v.size() && v[k + n] == v[k] + int32_t(n)) ++n;
                entries.push_back(make_int4(kind, v[k], int32_t(n), base + int32_t(k * unit)));
                k += n;
            }
        };
        auto add_spans = [&](const std::vector<int2>& v, int kind, int32_t base, size_t unit) {
            int64_t k = 0;
            for (const int2& sp : v) {
                entries.push_back(make_int4(kind, sp.x, sp.y, base + int32_t(k * int64_t(unit))));
                k += sp.y;
            }
        };
        add_runs(L.rows, ens::kMfsU, u_base, US);
        add_spans(L.uspan, ens::kMfsU, u_base + int32_t(L.rows.size() * US), US);
        add_spans(L.espan, ens::kMfsA, a_base, AS);
        add_runs(L.rows, ens::kMfsF, f_base, 32);
        entries.push_back(make_int4(ens::kMfsBlob, int32_t(blob.size() / 16), int32_t(L.blob_bytes), 0));
        t.n_entries = int32_t(entries.size()) - t.entry0;
        tiles.push_back(t);
        auto span_slot = [](const std::vector<int2>& v, int32_t q) -> int32_t {
            int32_t k = 0;
            for (const int2& sp : v) {
                if (q >= sp.x && q < sp.x + sp.y) return k + (q - sp.x);
                k += sp.y;
            }
            return -1;
        };
        auto uslot = [&](int32_t q) -> int32_t {
            auto it = std::lower_bound(L.rows.begin(), L.rows.end(), q);
            if (it != L.rows.end() && *it == q) return int32_t(it - L.rows.begin());
            return nr + span_slot(L.uspan, q);
        };
        auto eslot = [&](int32_t e) { return span_slot(L.espan, e); };
        size_t ninc = 0;
        for (int32_t r : L.rows) ninc += size_t(ip[size_t(r) + 1] - ip[size_t(r)]);
        std::vector<unsigned char> b(L.blob_bytes, 0);
        const int32_t roff = ens::kMfsHdrBytes + int32_t(ninc) * ens::kMfsRecBytes;
        const int32_t rid = roff + (nr + 1) * 4;
        const int32_t hdr[8] = {nr, u_base, roff, f_base, rid, 0, 0, 0};
        std::memcpy(b.data(), hdr, sizeof(hdr));
        int32_t q = 0;
        for (int32_t j = 0; j < nr; ++j) {
            const int32_t r = L.rows[size_t(j)];
            const int32_t o = q | int32_t(fx[size_t(r)]) << 24;
            std::memcpy(b.data() + roff + 4 * j, &o, 4);
            std::memcpy(b.data() + rid + 4 * j, &r, 4);
            for (int32_t k = ip[size_t(r)]; k < ip[size_t(r) + 1]; ++k, ++q) {
                const ens::FanRec& fr = rec[size_t(k)];
                const int32_t rc[4] = {a_base + eslot(fr.e) * int32_t(AS), u_base + uslot(fr.n_next) * int32_t(US),
                                       u_base + uslot(fr.n_prev) * int32_t(US), fr.restart};
                unsigned char* dst = b.data() + ens::kMfsHdrBytes + size_t(q) * ens::kMfsRecBytes;
                std::memcpy(dst, rc, 16);
                std::memcpy(dst + 16, k18.data() + size_t(k) * 18, 18 * sizeof(double));
            }
        }
        std::memcpy(b.data() + roff + 4 * nr, &q, 4);
        blob.insert(blob.end(), b.begin(), b.end());
    }
    if (blob.size() / 16 >= (size_t(1) << 31)) return fail(c, ENS_E_UNSUPPORTED, "matrix-free staged: tile blobs exceed 32 GB");
    out.row0 = row0;
    out.rows = rows;
    out.ntiles = int32_t(tiles.size());
    out.stage_bytes = sh.stage_bytes;
    RC_TRY(upload(c, &out.d_tiles, tiles.data(), tiles.size()));
    RC_TRY(upload(c, &out.d_entries, entries.data(), entries.size()));
    RC_TRY(upload(c, &out.d_blob, blob.data(), blob.size()));
    return ENS_OK;
}

int build_part(ens_ctx* c, Part& P, const Global& G) {
    const auto& pl = P.plan;
    const auto& pat = *G.pat;
    const int64_t n_s = c->n_s, lo = pl.lo, hi = pl.hi;
    P.n_own = hi - lo;
    P.n_gh = int64_t(pl.ghosts.size());
    const int64_t n_loc = P.n_own + P.n_gh;
    auto local = [&](int32_t g) -> int32_t {
        if (g >= lo && g < hi) return int32_t(g - lo);
        auto it = std::lower_bound(pl.ghosts.begin(), pl.ghosts.end(), g);
        return int32_t(P.n_own + (it - pl.ghosts.begin()));
    };
    // maps local row -> caller node id
    std::vector<int32_t> map_all(static_cast<size_t>(n_loc));
    for (int64_t i = 0; i < P.n_own; ++i) map_all[size_t(i)] = pat.perm[size_t(lo + i)];
    for (int64_t k = 0; k < P.n_gh; ++k) map_all[size_t(P.n_own + k)] = pat.perm[size_t(pl.ghosts[size_t(k)])];
    P.map_own.assign(map_all.begin(), map_all.begin() + P.n_own);
    // pattern of the owned rows, columns local, each row in its GLOBAL column order
    const int64_t b0 = pat.row_ptr[size_t(lo)], b1 = pat.row_ptr[size_t(hi)];
    std::vector<int32_t> rp(size_t(P.n_own) + 1), cl(size_t(b1 - b0));
    for (int64_t i = 0; i <= P.n_own; ++i) rp[size_t(i)] = int32_t(pat.row_ptr[size_t(lo + i)] - b0);
    for (int64_t b = b0; b < b1; ++b) cl[size_t(b - b0)] = local(pat.col[size_t(b)]);
    // coefficients of the owned rows
    std::vector<double> c1(size_t(P.n_own * n_s)), c2a, c3a;
    if (c->damping == ENS_DAMP_IDENTITY) { c2a.resize(c1.size()); c3a.resize(c1.size()); }
    const double dt = c->dt;
    for (int64_t i = 0; i < P.n_own; ++i)
        for (int64_t s = 0; s < n_s; ++s) {
            const double mi = (*G.mass)[size_t(s * c->V + map_all[size_t(i)])];
            const double cc = c->damping == ENS_DAMP_MASS ? c->c_d * mi : (c->damping == ENS_DAMP_IDENTITY ? c->c_d : 0.0);
            const double D = mi + 0.5 * dt * cc;
            c1[size_t(i * n_s + s)] = dt * dt / D;
            if (c->damping == ENS_DAMP_IDENTITY) {
                c2a[size_t(i * n_s + s)] = 2.0 * mi / D;
                c3a[size_t(i * n_s + s)] = (mi - 0.5 * dt * cc) / D;
            }
        }
    std::vector<uint8_t> fx(size_t(P.n_own), 0);
    if (G.fixed)
        for (int64_t i = 0; i < P.n_own; ++i) fx[size_t(i)] = G.fixed[map_all[size_t(i)]] & 7;
    RC_TRY(upload(c, &P.d_row_ptr, rp.data(), rp.size()));
    RC_TRY(upload(c, &P.d_col, cl.data(), cl.size()));
    RC_TRY(upload(c, &P.d_map_own, map_all.data(), size_t(P.n_own)));
    RC_TRY(upload(c, &P.d_map_all, map_all.data(), map_all.size()));
    if (c->multi) {            // one part per process: owned rows in local order (ens_get_owned)
        std::vector<int32_t> ident(size_t(P.n_own));
        for (int64_t i = 0; i < P.n_own; ++i) ident[size_t(i)] = int32_t(i);
        RC_TRY(upload(c, &P.d_map_abi, ident.data(), ident.size()));
    } else {
        P.d_map_abi = P.d_map_own;
    }
    RC_TRY(upload(c, &P.d_fixed, fx.data(), fx.size()));
    RC_TRY(upload(c, &P.d_c1, c1.data(), c1.size()));
    if (c->damping == ENS_DAMP_IDENTITY) {
        RC_TRY(upload(c, &P.d_c2a, c2a.data(), c2a.size()));
        RC_TRY(upload(c, &P.d_c3a, c3a.data(), c3a.size()));
    }
    if (!pl.send_rows.empty() && !c->p2p()) {
        RC_TRY(upload(c, &P.d_send_rows, pl.send_rows.data(), pl.send_rows.size()));
        RC_TRY(dalloc(c, &P.d_sendbuf, pl.send_rows.size() * 3 * size_t(n_s)));
    }
    // elements touching the owned rows -> local element ids
    std::vector<int32_t> elems;
    if (G.m->F) {
        std::vector<char> mark(size_t(G.m->F), 0);
        for (int64_t e = 0; e < G.m->F; ++e)
            for (int a = 0; a < 3; ++a) {
                int32_t g = pat.iperm[size_t(G.m->tris[3 * e + a])];
                if (g >= lo && g < hi) mark[size_t(e)] = 1;
            }
        if (c->kernel == ENS_KERNEL_MATRIX_FREE) {
            // matrix-free: elements numbered by first touch in row (fan) order, so that the
            // elements of consecutive rows are mostly consecutive (F3 copies alpha by runs)
            const ens::Fans& fans = *G.fans;
            for (int32_t k = fans.ptr[size_t(lo)]; k < fans.ptr[size_t(hi)]; ++k) {
                const int32_t e = fans.rec[size_t(k)].e;
                if (mark[size_t(e)] == 1) {
                    mark[size_t(e)] = 2;
                    elems.push_back(e);
                }
            }
        } else {
            for (int64_t e = 0; e < G.m->F; ++e)
                if (mark[size_t(e)]) elems.push_back(int32_t(e));
        }
    }
    std::vector<int32_t> eloc(size_t(G.m->F), -1);
    for (size_t k = 0; k < elems.size(); ++k) eloc[size_t(elems[k])] = int32_t(k);
    const int64_t Fl = int64_t(elems.size());
    std::vector<double> al(size_t(Fl * n_s));
    for (int64_t k = 0; k < Fl; ++k)
        for (int64_t s = 0; s < n_s; ++s) al[size_t(k * n_s + s)] = (*G.alpha)[size_t(s * G.m->F + elems[size_t(k)])];
    if (c->kernel == ENS_KERNEL_ASSEMBLED || c->kernel == ENS_KERNEL_ASSEMBLED_SYM) {
        // the global (full-CSR) blocks whose values this part stores
        std::vector<int64_t> blocks;
        if (c->kernel == ENS_KERNEL_ASSEMBLED) {
            for (int64_t b = b0; b < b1; ++b) blocks.push_back(b);
        } else {
            // half storage: row i keeps its blocks (i, j >= i); its blocks (i, j < i) are the
            // transposes of blocks (j, i), stored with row j if j is owned, else copied here
            std::vector<int32_t> lp(size_t(P.n_own) + 1, 0), li, lc, sc;
            std::vector<int2> ur(static_cast<size_t>(P.n_own));
            std::vector<int32_t> upper_at(size_t(b1 - b0), -1);
            auto find_block = [&](int32_t r, int32_t j) {
                auto first = pat.col.begin() + pat.row_ptr[size_t(r)];
                auto last = pat.col.begin() + pat.row_ptr[size_t(r) + 1];
                return int64_t(std::lower_bound(first, last, j) - pat.col.begin());
            };
            for (int64_t i = lo; i < hi; ++i) {
                for (int64_t b = pat.row_ptr[size_t(i)]; b < pat.row_ptr[size_t(i) + 1]; ++b) {
                    const int32_t j = pat.col[size_t(b)];
                    if (j >= i) continue;
                    int32_t idx;
                    if (j >= lo) {
                        idx = upper_at[size_t(find_block(j, int32_t(i)) - b0)];
                    } else {
                        idx = int32_t(blocks.size());
                        blocks.push_back(find_block(j, int32_t(i)));
                        sc.push_back(-1);
                    }
                    li.push_back(idx);
                    lc.push_back(local(j));
                }
                lp[size_t(i - lo) + 1] = int32_t(li.size());
                ur[size_t(i - lo)].x = int32_t(blocks.size());
                for (int64_t b = pat.row_ptr[size_t(i)]; b < pat.row_ptr[size_t(i) + 1]; ++b) {
                    const int32_t j = pat.col[size_t(b)];
                    if (j < i) continue;
                    upper_at[size_t(b - b0)] = int32_t(blocks.size());
                    blocks.push_back(b);
                    sc.push_back(local(j));
                }
                ur[size_t(i - lo)].y = int32_t(blocks.size());
            }
            RC_TRY(upload(c, &P.d_sym_lptr, lp.data(), lp.size()));
            RC_TRY(upload(c, &P.d_sym_lidx, li.data(), li.size()));
            RC_TRY(upload(c, &P.d_sym_lcol, lc.data(), lc.size()));
            RC_TRY(upload(c, &P.d_sym_urange, ur.data(), ur.size()));
            RC_TRY(upload(c, &P.d_sym_scol, sc.data(), sc.size()));
        }
        P.n_stored = int64_t(blocks.size());
        // F0 on the stored blocks: contributions re-indexed to local elements
        std::vector<int32_t> cp(blocks.size() + 1), cc;
        const auto& gcp = *G.contrib_ptr;
        const auto& gc = *G.contrib;
        for (size_t k = 0; k < blocks.size(); ++k) {
            cp[k] = int32_t(cc.size());
            for (int32_t q = gcp[size_t(blocks[k])]; q < gcp[size_t(blocks[k]) + 1]; ++q)
                cc.push_back(eloc[size_t(gc[size_t(q)] / 9)] * 9 + gc[size_t(q)] % 9);
        }
        cp[blocks.size()] = int32_t(cc.size());
        std::vector<double> kh(size_t(Fl) * 81);
        for (int64_t k = 0; k < Fl; ++k)
            std::copy_n(G.Khat->data() + size_t(elems[size_t(k)]) * 81, 81, kh.data() + size_t(k) * 81);
        int32_t *d_cp = nullptr, *d_cc = nullptr;
        double *d_al = nullptr, *d_kh = nullptr;
        RC_TRY(upload(c, &d_cp, cp.data(), cp.size()));
        RC_TRY(upload(c, &d_cc, cc.data(), cc.size()));
        RC_TRY(upload(c, &d_al, al.data(), al.size()));
        RC_TRY(upload(c, &d_kh, kh.data(), kh.size()));
        RC_TRY(dalloc(c, &P.d_Kval, blocks.size() * 9 * size_t(n_s)));
        CUDA_TRY(c, ens::launch_assemble(int64_t(blocks.size()), c->n_s, d_cp, d_cc, d_al, d_kh, P.d_Kval, c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        dfree(c, d_kh);
        if (c->reassemble_every > 0) {          // keep what the geometry-updated rebuild needs
            std::vector<int32_t> et(size_t(Fl) * 3);
            for (int64_t k = 0; k < Fl; ++k)
                for (int a = 0; a < 3; ++a)
                    et[size_t(3 * k + a)] = local(pat.iperm[size_t(G.m->tris[3 * int64_t(elems[size_t(k)]) + a])]);
            std::vector<double> xl(size_t(n_loc) * 3);
            for (int64_t r = 0; r < n_loc; ++r)
                for (int d = 0; d < 3; ++d) xl[size_t(3 * r + d)] = G.m->xyz[3 * int64_t(map_all[size_t(r)]) + d];
            RC_TRY(upload(c, &P.d_retri, et.data(), et.size()));
            RC_TRY(upload(c, &P.d_rxyz, xl.data(), xl.size()));
            P.d_rcp = d_cp;
            P.d_rcc = d_cc;
            P.d_ral = d_al;
        } else {
            dfree(c, d_cp);
            dfree(c, d_cc);
            dfree(c, d_al);
        }
    } else {
        const ens::Fans& fans = *G.fans;
        const int32_t k0 = fans.ptr[size_t(lo)], k1 = fans.ptr[size_t(hi)];
        std::vector<int32_t> ip(size_t(P.n_own) + 1);
        for (int64_t i = 0; i <= P.n_own; ++i) ip[size_t(i)] = fans.ptr[size_t(lo + i)] - k0;
        std::vector<ens::FanRec> rec(fans.rec.begin() + k0, fans.rec.begin() + k1);
        for (auto& r : rec) {
            r.e = eloc[size_t(r.e)];
            r.n_prev = local(r.n_prev);
            r.n_next = local(r.n_next);
        }
        const int Pg = c->n_s / ens::pick_vec_mf(c->n_s);
        P.mf_groups = std::min(Pg, 256);
        P.mf_rows = std::max(1, std::min(256 / P.mf_groups, 32));
        // launch_rows tiles [row0, row0 + rows) from row0: the whole range (no halo), and with
        // a halo the boundary ranges [0, b_lo), [n_own - b_hi, n_own) and the interior
        // [b_lo, n_own - b_hi) — every tiling launched sizes the shared-memory image
        std::vector<std::pair<int64_t, int64_t>> tilings = {{0, P.n_own}};
        if (pl.b_lo || pl.b_hi)
            tilings.insert(tilings.end(), {{0, pl.b_lo}, {P.n_own - pl.b_hi, P.n_own}, {pl.b_lo, P.n_own - pl.b_hi}});
        for (;;) {
            int32_t mx = 0;
            for (const auto& tl : tilings)
                for (int64_t r0 = tl.first; r0 < tl.second; r0 += P.mf_rows) {
                    const int64_t r1 = std::min<int64_t>(r0 + P.mf_rows, tl.second);
                    mx = std::max(mx, ip[size_t(r1)] - ip[size_t(r0)]);
                }
            P.mf_smem_inc = mx;
            if (int64_t(mx) * ens::mf_inc_bytes() <= 96 * 1024 || P.mf_rows == 1) break;
            P.mf_rows = std::max(1, P.mf_rows / 2);
        }
        if (c->mf_variant == ENS_MF_TILES && int64_t(P.mf_smem_inc) * ens::mf_inc_bytes() > 200 * 1024)
            return fail(c, ENS_E_UNSUPPORTED, "a node has too many incident elements for the matrix-free kernel");
        static_assert(sizeof(ens::FanRec) == sizeof(int4), "FanRec layout");
        std::vector<std::vector<std::vector<int32_t>>> patches;     // F3: per launched range
        if (c->mf_variant == ENS_MF_STAGED) {
            const ens::MfsShape sh = ens::mf_staged_shape(c->mfs_plan.shape);
            const size_t W = size_t(ens::mfs_stage_w(c->mfs_plan, n_s));
            const size_t US = W * 24, AS = W * 8;
            for (const auto& tl : tilings)
                patches.push_back(tl.second > tl.first
                                      ? mf_patches(ip, rec, n_loc, tl.first, tl.second - tl.first, US, AS, mfs_budget(c, sh), c->mfs_plan)
                                      : std::vector<std::vector<int32_t>>());
            // elements renumbered by first touch in the (whole-range) tile order: each tile's
            // alpha rows then move in few runs
            std::vector<int32_t> new_of(static_cast<size_t>(Fl), -1);
            int32_t next = 0;
            for (const auto& tile : patches[0]) {
                std::vector<int32_t> rs(tile);
                std::sort(rs.begin(), rs.end());
                for (int32_t r : rs)
                    for (int32_t k = ip[size_t(r)]; k < ip[size_t(r) + 1]; ++k)
                        if (new_of[size_t(rec[size_t(k)].e)] < 0) new_of[size_t(rec[size_t(k)].e)] = next++;
            }
            for (auto& x : new_of)
                if (x < 0) x = next++;
            std::vector<double> al2(al.size());
            for (int64_t e = 0; e < Fl; ++e)
                std::copy_n(al.data() + size_t(e) * size_t(n_s), n_s, al2.data() + size_t(new_of[size_t(e)]) * size_t(n_s));
            al.swap(al2);
            for (auto& r : rec) r.e = new_of[size_t(r.e)];
        }
        RC_TRY(upload(c, &P.d_inc_ptr, ip.data(), ip.size()));
        RC_TRY(upload(c, &P.d_fan, reinterpret_cast<const int4*>(rec.data()), rec.size()));
        if (ens::mf_diff()) {      // (prev, next) columns only: K^_e[a,a] u_i cancels (kernels.cu DIFF)
            std::vector<double> k18(size_t(k1 - k0) * 18);
            for (int64_t k = 0; k < k1 - k0; ++k)
                for (int c = 0; c < 3; ++c)
                    for (int b = 0; b < 2; ++b)
                        for (int d = 0; d < 3; ++d)
                            k18[size_t(k) * 18 + size_t(6 * c + 3 * b + d)] =
                                fans.Krow[size_t(k0 + k) * 28 + size_t(9 * c + 3 * (b + 1) + d)];
            RC_TRY(upload(c, &P.d_Krow, k18.data(), k18.size()));
            // item programs of the per-warp streaming kernel (kernels.cu F2w): per row
            // OWN, then per incidence [PREV at a chain start] INC, then OLD
            std::vector<int32_t> iptr(size_t(P.n_own) + 1);
            std::vector<int4> items;
            items.reserve(size_t(P.n_own) * 2 + rec.size() * 2);
            for (int64_t i = 0; i < P.n_own; ++i) {
                iptr[size_t(i)] = int32_t(items.size());
                const int32_t kb = ip[size_t(i)], ke = ip[size_t(i) + 1];
                const int32_t ii = int32_t(i);
                items.push_back(make_int4(ii, ii, 0, ens::kItemOwn | (kb == ke ? ens::kItemLastApply : 0)));
                for (int32_t k = kb; k < ke; ++k) {
                    const ens::FanRec& r = rec[size_t(k)];
                    if (k == kb || r.restart) items.push_back(make_int4(r.n_prev, ii, 0, ens::kItemPrev));
                    items.push_back(make_int4(r.n_next, r.e, k, ens::kItemInc | (k + 1 == ke ? ens::kItemLastApply : 0)));
                }
                items.push_back(make_int4(ii, ii, 0, ens::kItemOld | (int32_t(fx[size_t(i)]) << 8)));
            }
            iptr[size_t(P.n_own)] = int32_t(items.size());
            if (c->mf_variant == ENS_MF_WARP) {
                RC_TRY(upload(c, &P.d_item_ptr, iptr.data(), iptr.size()));
                RC_TRY(upload(c, &P.d_items, items.data(), items.size()));
            }
            if (c->mf_variant == ENS_MF_STAGED)
                for (size_t q = 0; q < tilings.size(); ++q) {
                    if (tilings[q].second <= tilings[q].first) continue;
                    P.mfs.emplace_back();
                    RC_TRY(build_mf_tiles(c, ip, rec, k18, fx, patches[q], tilings[q].first,
                                          tilings[q].second - tilings[q].first, P.mfs.back()));
                }
        } else {
            RC_TRY(upload(c, &P.d_Krow, fans.Krow.data() + size_t(k0) * 28, size_t(k1 - k0) * 28));
        }
        RC_TRY(upload(c, &P.d_alpha, al.data(), al.size()));
        P.n_alpha = Fl;
    }
    const size_t ns = size_t(n_loc) * 3 * size_t(n_s);
    if (c->multi && c->p2p()) {      // exported to the neighbours: plain cudaMalloc (IPC)
        RC_TRY(rawalloc(c, &P.d_u0, ns));
        RC_TRY(rawalloc(c, &P.d_u1, ns));
    } else {
        RC_TRY(dalloc(c, &P.d_u0, ns));
        RC_TRY(dalloc(c, &P.d_u1, ns));
    }
    CUDA_TRY(c, cudaMemsetAsync(P.d_u0, 0, ns * sizeof(double), c->stream));
    CUDA_TRY(c, cudaMemsetAsync(P.d_u1, 0, ns * sizeof(double), c->stream));
    return ENS_OK;
}

// P2P halo tables of part P (rank p) from every part's plan: send row send_rows[off + j]
// to neighbour q lands in q's local row recv_row(q <- p) + j (q's ghosts are sorted, and
// those owned by p are contiguous there); q's flags[p] is where p publishes its steps.
int build_p2p(ens_ctx* c, Part& P, const std::vector<ens::PartPlan>& plans) {
    const auto& pl = P.plan;
    const int32_t p = pl.p;
    std::vector<std::vector<int2>> dst(static_cast<size_t>(P.n_own));
    std::vector<int32_t> in_q;
    for (const auto& pe : pl.peers) {
        if (pe.recv_n) in_q.push_back(pe.q);
        if (!pe.send_n) continue;
        const ens::PartPlan& Q = plans[size_t(pe.q)];
        const auto it = std::find_if(Q.peers.begin(), Q.peers.end(), [&](const ens::PartPlan::Peer& x) { return x.q == p; });
        if (it == Q.peers.end() || it->recv_n != pe.send_n)
            return fail(c, ENS_E_ARG, "P2P halo: inconsistent plans of parts " + std::to_string(p) + " and " +
                                          std::to_string(pe.q));
        const int32_t slot = int32_t(P.out_q.size());
        P.out_q.push_back(pe.q);
        P.out_rows.push_back(Q.n_own() + int64_t(Q.ghosts.size()));
        for (int64_t j = 0; j < pe.send_n; ++j)
            dst[size_t(pl.send_rows[size_t(pe.send_off + j)])].push_back(make_int2(slot, int32_t(it->recv_row + j)));
    }
    std::vector<int32_t> fptr(size_t(P.n_own) + 1, 0);
    std::vector<int2> fdst;
    for (int64_t i = 0; i < P.n_own; ++i) {
        for (const int2& d : dst[size_t(i)]) fdst.push_back(d);
        fptr[size_t(i) + 1] = int32_t(fdst.size());
    }
    P.n_out = int32_t(P.out_q.size());
    P.n_in = int32_t(in_q.size());
    RC_TRY(upload(c, &P.d_fwd_ptr, fptr.data(), fptr.size()));
    RC_TRY(upload(c, &P.d_fwd_dst, fdst.data(), fdst.size()));
    RC_TRY(upload(c, &P.d_in_q, in_q.data(), in_q.size()));
    RC_TRY(dalloc(c, &P.d_hdone, 1));
    CUDA_TRY(c, cudaMemsetAsync(P.d_hdone, 0, sizeof(unsigned int), c->stream));
    RC_TRY(dalloc(c, &P.d_peer_buf, size_t(2 * P.n_out)));
    RC_TRY(dalloc(c, &P.d_out_flag, size_t(P.n_out)));
    const size_t nf = size_t(c->world);
    if (c->multi) RC_TRY(rawalloc(c, &P.d_hflags, nf));
    else RC_TRY(dalloc(c, &P.d_hflags, nf));
    CUDA_TRY(c, cudaMemsetAsync(P.d_hflags, 0, nf * sizeof(unsigned long long), c->stream));
    return ENS_OK;
}

// emulation (all parts here): the neighbours' tables are this context's own parts
int link_p2p_local(ens_ctx* c) {
    for (Part& P : c->parts) {
        std::vector<double*> pb;
        std::vector<unsigned long long*> of;
        for (int32_t q : P.out_q) {
            Part& Q = c->parts[size_t(q)];
            pb.push_back(Q.d_u0);
            pb.push_back(Q.d_u1);
            of.push_back(Q.d_hflags + P.plan.p);
        }
        if (!pb.empty()) {
            CUDA_TRY(c, cudaMemcpyAsync(P.d_peer_buf, pb.data(), pb.size() * sizeof(double*), cudaMemcpyHostToDevice,
                                        c->stream));
            CUDA_TRY(c, cudaMemcpyAsync(P.d_out_flag, of.data(), of.size() * sizeof(void*), cudaMemcpyHostToDevice,
                                        c->stream));
        }
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return ENS_OK;
}

int finish_create(ens_ctx* c) {
    RC_TRY(dalloc(c, &c->d_stage, size_t(c->V) * 3 * size_t(c->n_s)));
    RC_TRY(dalloc(c, &c->d_flag, 1));
    RC_TRY(dalloc(c, &c->d_herr, 1));
    RC_TRY(dalloc(c, &c->d_coef, 2 * ens::kMaxFields));
    c->coef_dirty = true;
    RC_TRY(dalloc(c, &c->d_step, 1));
    CUDA_TRY(c, cudaMemsetAsync(c->d_flag, 0xff, sizeof(unsigned long long), c->stream));
    CUDA_TRY(c, cudaMemsetAsync(c->d_herr, 0xff, sizeof(unsigned long long), c->stream));
    CUDA_TRY(c, cudaMemsetAsync(c->d_step, 0, sizeof(int64_t), c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    c->step = 0;
    return ENS_OK;
}

int create_impl(ens_ctx* c, const ens_mesh* mesh, const ens_materials* mat, const ens_options* opt) {
    const int64_t V = mesh->n_nodes, F = mesh->n_tris, NV = int64_t(mat->n_s) * V;
    ens::MeshView m{V, F, mesh->xyz, mesh->tris};
    RC_TRY(init_ctx(c, opt));
    c->V = V;
    c->F = F;
    c->n_s = mat->n_s;
    c->s_begin = mat->s_begin;
    if (c->kernel == ENS_KERNEL_MATRIX_FREE) {        // the data path (ens.h ENS_MF_*)
        const int32_t req = opt ? opt->mf_variant : int32_t(ENS_MF_AUTO);
        const bool diff = ens::mf_diff();
        const bool staged_ok = diff && ens::mf_staged_applies(c->n_s);
        const bool warp_ok = diff && c->n_s % 64 == 0 && c->damping != ENS_DAMP_IDENTITY;
        if (req == ENS_MF_AUTO) c->mf_variant = staged_ok ? ENS_MF_STAGED : ENS_MF_TILES;
        else if (req == ENS_MF_STAGED && !staged_ok)
            return fail(c, ENS_E_UNSUPPORTED, "mf_variant STAGED needs an even n_s >= 64 (and the DIFF form)");
        else if (req == ENS_MF_WARP && !warp_ok)
            return fail(c, ENS_E_UNSUPPORTED, "mf_variant WARP needs n_s % 64 == 0 and damping != IDENTITY");
        else c->mf_variant = req;
        c->mfs_plan = ens::mf_staged_plan(c->n_s);
    }

    // S0: pattern (RCM + block CSR)
    ens::Pattern pat = ens::build_pattern(m);
    c->nnzb = int64_t(pat.col.size());
    c->bandwidth = pat.bandwidth;
    c->perm = pat.perm;
    c->iperm = pat.iperm;
    if (c->nnzb >= (int64_t(1) << 31)) return fail(c, ENS_E_ARG, "pattern exceeds 2^31 blocks");

    // S1: element stiffness, Gauss-point scaling, mass, CFL
    std::vector<double> Khat(size_t(81 * F)), area(static_cast<size_t>(F));
    for (int64_t e = 0; e < F; ++e)
        ens::element_stiffness(mesh->xyz + 3 * int64_t(mesh->tris[3 * e]), mesh->xyz + 3 * int64_t(mesh->tris[3 * e + 1]),
                               mesh->xyz + 3 * int64_t(mesh->tris[3 * e + 2]), mat->nu, mat->k_shear,
                               Khat.data() + 81 * e, area.data() + e);
    std::vector<double> alpha(size_t(mat->n_s * F)), mass(static_cast<size_t>(NV));
    ens::materials(m, mat->n_s, mat->E, mat->h, mat->rho, alpha.data(), mass.data());
    const double safety = (opt && opt->cfl_safety > 0.0) ? opt->cfl_safety : 0.9;
    c->dt_cfl = ens::cfl_dt(m, mat->n_s, mat->E, mat->rho, safety);
    c->dt = (opt && opt->dt > 0.0) ? opt->dt : c->dt_cfl;
    if (c->damping == ENS_DAMP_MASS) {       // C~ = c_d M~: c2, c3 independent of the node
        const double q = 0.5 * c->dt * c->c_d;
        c->c2 = 2.0 / (1.0 + q);
        c->c3 = (1.0 - q) / (1.0 + q);
    }

    // element -> block contributions (assembled) or fans (matrix-free), global
    std::vector<int32_t> cptr, contrib;
    ens::Fans fans;
    if (c->kernel != ENS_KERNEL_MATRIX_FREE) {
        cptr.assign(size_t(c->nnzb) + 1, 0);
        contrib.resize(size_t(9 * F));
        std::vector<int32_t> blk(size_t(9 * F));
        for (int64_t e = 0; e < F; ++e)
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) {
                    const int32_t i = pat.iperm[size_t(mesh->tris[3 * e + a])], j = pat.iperm[size_t(mesh->tris[3 * e + b])];
                    auto first = pat.col.begin() + pat.row_ptr[size_t(i)];
                    auto last = pat.col.begin() + pat.row_ptr[size_t(i) + 1];
                    const int32_t bi = int32_t(std::lower_bound(first, last, j) - pat.col.begin());
                    blk[size_t(9 * e + 3 * a + b)] = bi;
                    cptr[size_t(bi) + 1]++;
                }
        for (size_t k = 1; k < cptr.size(); ++k) cptr[k] += cptr[k - 1];
        std::vector<int32_t> fillp(cptr.begin(), cptr.end() - 1);
        for (int64_t e = 0; e < F; ++e)                   // ascending e => ascending within a block
            for (int ab = 0; ab < 9; ++ab) contrib[size_t(fillp[size_t(blk[size_t(9 * e + ab)])]++)] = int32_t(9 * e + ab);
    } else {
        fans = ens::build_fans(m, pat.iperm, Khat);
        if (c->mf_variant == ENS_MF_STAGED) {
            // every single row's stage image must fit (own + neighbour u rows, alpha rows,
            // records, F_k): at large N_s a high-degree node may not; AUTO then falls back to
            // TILES, an explicit STAGED request fails
            const ens::MfsShape sh = ens::mf_staged_shape(c->mfs_plan.shape);
            const size_t W = size_t(ens::mfs_stage_w(c->mfs_plan, c->n_s));
            const size_t US = W * 24, AS = W * 8;
            size_t worst = 0;
            std::vector<int32_t> nb;
            for (int64_t i = 0; i < V; ++i) {
                nb.clear();
                for (int32_t k = fans.ptr[size_t(i)]; k < fans.ptr[size_t(i) + 1]; ++k) {
                    nb.push_back(fans.rec[size_t(k)].n_prev);
                    nb.push_back(fans.rec[size_t(k)].n_next);
                }
                std::sort(nb.begin(), nb.end());
                const size_t nn = size_t(std::unique(nb.begin(), nb.end()) - nb.begin());
                const size_t ninc = size_t(fans.ptr[size_t(i) + 1] - fans.ptr[size_t(i)]);
                const size_t blob = (size_t(ens::kMfsHdrBytes) + ninc * ens::kMfsRecBytes + 12 + 127) & ~size_t(127);
                worst = std::max(worst, blob + (1 + nn) * US + ninc * AS + size_t(ens::kMaxFields) * 32);
            }
            if (worst > mfs_budget(c, sh)) {
                if (!opt || opt->mf_variant == ENS_MF_AUTO) c->mf_variant = ENS_MF_TILES;
                else return fail(c, ENS_E_UNSUPPORTED, "mf_variant STAGED: one row's operands (" + std::to_string(worst) +
                                                          " B) exceed a shared-memory stage at this N_s");
            }
        }
    }

    // partitions: one part unless node-partitioned; all parts here unless NCCL is used
    const int32_t P = c->dist == ENS_DIST_NODE ? c->world : 1;
    std::vector<ens::PartPlan> plans = P > 1 ? ens::halo_plan(pat.row_ptr, pat.col, P)
                                             : std::vector<ens::PartPlan>(1);
    if (P == 1) {
        plans[0].lo = 0;
        plans[0].hi = V;
    }
    Global G{&m, &pat, &Khat, &alpha, &mass, mesh->fixed, &fans, &cptr, &contrib};
    if (c->multi && P > 1) {
        c->parts.resize(1);
        c->parts[0].plan = plans[size_t(c->rank)];
    } else {
        c->parts.resize(plans.size());
        for (size_t k = 0; k < plans.size(); ++k) c->parts[k].plan = plans[k];
    }
    for (Part& p : c->parts) RC_TRY(build_part(c, p, G));
    if (c->has_halo() && !c->comm_stream) {      // the halo chain's stream (one-context emulation)
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_packed, cudaEventDisableTiming));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
    }
    if (c->p2p()) {
        for (Part& p : c->parts) RC_TRY(build_p2p(c, p, plans));
        if (!c->multi) RC_TRY(link_p2p_local(c));
    }
    // element means of E per realisation (stress recovery, ens_stress)
    c->h_xyz.assign(mesh->xyz, mesh->xyz + 3 * V);
    c->h_tris.assign(mesh->tris, mesh->tris + 3 * F);
    c->nu = mat->nu;
    c->k_shear = mat->k_shear;
    {
        std::vector<double> eb(size_t(F) * size_t(mat->n_s));
        for (int64_t e = 0; e < F; ++e)
            for (int64_t s = 0; s < mat->n_s; ++s) {
                const double* Es = mat->E + s * V;
                eb[size_t(e * mat->n_s + s)] =
                    (Es[mesh->tris[3 * e]] + Es[mesh->tris[3 * e + 1]] + Es[mesh->tris[3 * e + 2]]) / 3.0;
            }
        RC_TRY(upload(c, &c->d_Ebar, eb.data(), eb.size()));
    }
    return finish_create(c);
}

int arg_check(const ens_mesh* mesh, const ens_materials* mat) {
    if (!mesh || !mat) return fail(nullptr, ENS_E_ARG, "mesh or materials is NULL");
    if (mesh->n_nodes < 1 || mesh->n_tris < 1 || !mesh->xyz || !mesh->tris)
        return fail(nullptr, ENS_E_ARG, "mesh needs n_nodes >= 1, n_tris >= 1, xyz and tris");
    if (mesh->n_nodes >= (int64_t(1) << 31) || 9 * mesh->n_tris >= (int64_t(1) << 31))
        return fail(nullptr, ENS_E_ARG, "mesh too large for 32-bit node / element ids");
    if (mat->n_s < 1 || !mat->E || !mat->h) return fail(nullptr, ENS_E_ARG, "materials need n_s >= 1, E and h");
    if (mat->n_s >= (1 << 24)) return fail(nullptr, ENS_E_ARG, "n_s must be < 2^24");
    if (!(mat->rho > 0.0) || !std::isfinite(mat->rho)) return fail(nullptr, ENS_E_ARG, "rho must be > 0");
    if (!(mat->nu >= 0.0 && mat->nu <= 0.5)) return fail(nullptr, ENS_E_ARG, "nu must lie in [0, 0.5]");
    if (!(mat->k_shear > 0.0) || !std::isfinite(mat->k_shear)) return fail(nullptr, ENS_E_ARG, "k_shear must be > 0");
    const int64_t V = mesh->n_nodes, NV = int64_t(mat->n_s) * V;
    for (int64_t k = 0; k < NV; ++k) {
        if (!(mat->E[k] > 0.0) || !std::isfinite(mat->E[k]))
            return fail(nullptr, ENS_E_ARG, "E[" + std::to_string(k / V) + "][" + std::to_string(k % V) + "] must be finite and > 0");
        if (!(mat->h[k] > 0.0) || !std::isfinite(mat->h[k]))
            return fail(nullptr, ENS_E_ARG, "h[" + std::to_string(k / V) + "][" + std::to_string(k % V) + "] must be finite and > 0");
    }
    ens::MeshView m{V, mesh->n_tris, mesh->xyz, mesh->tris};
    int64_t bad = -1;
    const int vcode = ens::validate_mesh(m, &bad);
    if (vcode) {
        static const char* what[] = {"", "node index out of range in element ", "repeated node in element ",
                                     "degenerate (zero-area) element ", "edge shared by more than two triangles at node ",
                                     "node in no triangle (zero lumped mass): node "};
        return fail(nullptr, ENS_E_MESH, std::string(what[vcode]) + std::to_string(bad));
    }
    return ENS_OK;
}

}  // namespace

extern "C" {

int ens_create(const ens_mesh* mesh, const ens_materials* mat, const ens_options* opt, ens_ctx** out) {
    if (!out) return fail(nullptr, ENS_E_ARG, "out is NULL");
    *out = nullptr;
    RC_TRY(arg_check(mesh, mat));
    RC_TRY(check_opts(opt));
    ens_ctx* c = new ens_ctx();
    const int rc = create_impl(c, mesh, mat, opt);
    if (rc) {
        const std::string msg = c->err;
        free_all(c);
        delete c;
        g_err = msg;
        return rc;
    }
    *out = c;
    return ENS_OK;
}

int ens_create_csr(int64_t n_nodes, const int64_t* row_ptr, const int32_t* col, int32_t n_s, const double* Kval,
                   const double* c1, const double* c2, const double* c3, const uint8_t* fixed, double dt,
                   const ens_options* opt, ens_ctx** out) {
    if (!out) return fail(nullptr, ENS_E_ARG, "out is NULL");
    *out = nullptr;
    if (n_nodes < 1 || !row_ptr || !col || n_s < 1 || !Kval || !c1 || !c2 || !c3)
        return fail(nullptr, ENS_E_ARG, "ens_create_csr: bad arguments");
    RC_TRY(check_opts(opt));
    if (opt && (opt->kernel != ENS_KERNEL_ASSEMBLED || opt->dist == ENS_DIST_NODE))
        return fail(nullptr, ENS_E_ARG, "ens_create_csr needs kernel = ASSEMBLED, dist != NODE");
    const int64_t V = n_nodes, nnzb = row_ptr[V];
    for (int64_t i = 0; i < V; ++i)
        if (row_ptr[i + 1] < row_ptr[i]) return fail(nullptr, ENS_E_ARG, "row_ptr not monotone");
    for (int64_t b = 0; b < nnzb; ++b)
        if (col[b] < 0 || col[b] >= V) return fail(nullptr, ENS_E_ARG, "column index out of range");
    ens_ctx* c = new ens_ctx();
    auto body = [&]() -> int {
        RC_TRY(init_ctx(c, opt));
        c->kernel = ENS_KERNEL_ASSEMBLED;
        c->damping = ENS_DAMP_IDENTITY;      // arbitrary per-DOF c2, c3 arrays
        c->reassemble_every = 0;             // no geometry behind a synthetic operator
        c->V = V;
        c->F = 0;
        c->nnzb = nnzb;
        c->n_s = n_s;
        c->dt = c->dt_cfl = dt;
        c->perm.resize(size_t(V));
        for (int64_t i = 0; i < V; ++i) c->perm[size_t(i)] = int32_t(i);
        c->iperm = c->perm;
        c->parts.resize(1);
        Part& P = c->parts[0];
        P.plan.lo = 0;
        P.plan.hi = V;
        P.n_own = V;
        P.map_own = c->perm;
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
        RC_TRY(upload(c, &P.d_row_ptr, rp32.data(), rp32.size()));
        RC_TRY(upload(c, &P.d_col, col, size_t(nnzb)));
        RC_TRY(upload(c, &P.d_map_own, c->perm.data(), c->perm.size()));
        RC_TRY(upload(c, &P.d_map_all, c->perm.data(), c->perm.size()));
        P.d_map_abi = P.d_map_own;
        RC_TRY(upload(c, &P.d_fixed, fx.data(), fx.size()));
        RC_TRY(upload(c, &P.d_Kval, kv.data(), kv.size()));
        RC_TRY(upload(c, &P.d_c1, a1.data(), a1.size()));
        RC_TRY(upload(c, &P.d_c2a, a2.data(), a2.size()));
        RC_TRY(upload(c, &P.d_c3a, a3.data(), a3.size()));
        const size_t ns = size_t(V) * 3 * size_t(n_s);
        RC_TRY(dalloc(c, &P.d_u0, ns));
        RC_TRY(dalloc(c, &P.d_u1, ns));
        CUDA_TRY(c, cudaMemsetAsync(P.d_u0, 0, ns * sizeof(double), c->stream));
        CUDA_TRY(c, cudaMemsetAsync(P.d_u1, 0, ns * sizeof(double), c->stream));
        return finish_create(c);
    };
    const int rc = body();
    if (rc) {
        const std::string msg = c->err;
        free_all(c);
        delete c;
        g_err = msg;
        return rc;
    }
    *out = c;
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
    // Same shape as the current traction: pack into the pinned staging and enqueue the
    // copies on the stream (they run after the steps already enqueued), no synchronisation
    // and no graph rebuild — the per-window input update of a running simulation.
    size_t need = size_t(n_tab) * size_t(1 + n_fields);
    for (const Part& p : c->parts) need += size_t(n_fields) * size_t(p.n_own) * 4;
    if (n_fields > 0 && n_fields == c->n_fields && n_tab == c->n_tab && c->h_trac && c->h_trac_n == need) {
        CUDA_TRY(c, cudaEventSynchronize(c->ev_trac));  // the previous update has left the staging
        double* h = c->h_trac;
        for (Part& p : c->parts) {
            double* Fd = h;
            for (int32_t k = 0; k < n_fields; ++k)
                for (int64_t i = 0; i < p.n_own; ++i) {
                    double* dst = Fd + (k * p.n_own + i) * 4;
                    const double* src = F + (k * c->V + p.map_own[size_t(i)]) * 3;
                    dst[0] = src[0];
                    dst[1] = src[1];
                    dst[2] = src[2];
                    dst[3] = 0.0;
                }
            const size_t nb = size_t(n_fields) * size_t(p.n_own) * 4;
            CUDA_TRY(c, cudaMemcpyAsync(p.d_Fk, Fd, nb * sizeof(double), cudaMemcpyHostToDevice, c->stream));
            h += nb;
        }
        if (n_tab > 0) {
            std::copy(tab_t, tab_t + n_tab, h);
            std::copy(tab_g, tab_g + size_t(n_tab) * size_t(n_fields), h + n_tab);
            CUDA_TRY(c, cudaMemcpyAsync(c->d_tab_t, h, size_t(n_tab) * sizeof(double), cudaMemcpyHostToDevice,
                                        c->stream));
            CUDA_TRY(c, cudaMemcpyAsync(c->d_tab_g, h + n_tab, size_t(n_tab) * size_t(n_fields) * sizeof(double),
                                        cudaMemcpyHostToDevice, c->stream));
        }
        CUDA_TRY(c, cudaEventRecord(c->ev_trac, c->stream));
        if (period != c->period || ramp_T != c->ramp_T) drop_graph(c);   // scalars of the captured steps
        c->period = period;
        c->ramp_T = ramp_T;
        c->coef_dirty = true;
        return ENS_OK;
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));       // old buffers may still be in use
    drop_graph(c);
    c->n_fields = 0;
    c->n_tab = 0;
    dfree(c, c->d_tab_t);
    dfree(c, c->d_tab_g);
    for (Part& p : c->parts) {
        dfree(c, p.d_Fk);
        std::vector<double> Fd(size_t(n_fields * p.n_own * 4), 0.0);     // [k][row][4]
        for (int32_t k = 0; k < n_fields; ++k)
            for (int64_t i = 0; i < p.n_own; ++i)
                for (int d = 0; d < 3; ++d)
                    Fd[size_t((k * p.n_own + i) * 4 + d)] = F[(k * c->V + p.map_own[size_t(i)]) * 3 + d];
        RC_TRY(upload(c, &p.d_Fk, Fd.data(), Fd.size()));
    }
    if (n_tab > 0) {
        RC_TRY(upload(c, &c->d_tab_t, tab_t, size_t(n_tab)));
        RC_TRY(upload(c, &c->d_tab_g, tab_g, size_t(n_tab) * size_t(n_fields)));
    }
    c->n_fields = n_fields;
    c->n_tab = n_tab;
    c->period = period;
    c->ramp_T = ramp_T;
    c->coef_dirty = true;
    // pinned staging for later same-shape updates
    if (c->h_trac) cudaFreeHost(c->h_trac);
    c->h_trac = nullptr;
    c->h_trac_n = 0;
    if (need > 0) {
        CUDA_TRY(c, cudaHostAlloc(reinterpret_cast<void**>(&c->h_trac), need * sizeof(double), cudaHostAllocDefault));
        c->h_trac_n = need;
        if (!c->ev_trac) CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_trac, cudaEventDisableTiming));
        CUDA_TRY(c, cudaEventRecord(c->ev_trac, c->stream));
    }
    return ENS_OK;
}

int ens_observe(ens_ctx* c, double* u_n) {
    if (!c || !u_n) return fail(c, ENS_E_ARG, "NULL argument");
    if (!c->obs_stream) {
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->obs_stream, cudaStreamNonBlocking));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_obs_ready, cudaEventDisableTiming));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->ev_obs_done, cudaEventDisableTiming));
        CUDA_TRY(c, cudaHostAlloc(reinterpret_cast<void**>(&c->h_obs_flag), sizeof(unsigned long long),
                                  cudaHostAllocDefault));
        const int64_t rows = c->multi ? c->parts[0].n_own : c->V;
        RC_TRY(dalloc(c, &c->d_obs, size_t(rows) * 3 * size_t(c->n_s)));
    }
    const int64_t Vabi = c->multi ? c->parts[0].n_own : c->V;
    if (c->obs_pending) CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->ev_obs_done, 0));   // d_obs is free
    for (Part& p : c->parts) {
        const double* src = (c->step & 1) ? p.d_u1 : p.d_u0;     // u_n = buf[step & 1]
        CUDA_TRY(c, ens::launch_dev_to_abi(p.n_own, c->n_s, p.d_map_abi, Vabi, src, c->d_obs, c->stream));
    }
    CUDA_TRY(c, cudaEventRecord(c->ev_obs_ready, c->stream));
    CUDA_TRY(c, cudaStreamWaitEvent(c->obs_stream, c->ev_obs_ready, 0));
    CUDA_TRY(c, cudaMemcpyAsync(u_n, c->d_obs, size_t(Vabi) * 3 * size_t(c->n_s) * sizeof(double),
                                cudaMemcpyDeviceToHost, c->obs_stream));
    CUDA_TRY(c, cudaMemcpyAsync(c->h_obs_flag, c->d_flag, sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                c->obs_stream));
    CUDA_TRY(c, cudaEventRecord(c->ev_obs_done, c->obs_stream));
    c->obs_pending = true;
    c->obs_step = c->step;
    return ENS_OK;
}

int ens_observe_wait(ens_ctx* c, int64_t* step) {
    if (!c) return fail(nullptr, ENS_E_ARG, "ctx is NULL");
    if (!c->obs_pending) return fail(c, ENS_E_STATE, "no snapshot in flight (call ens_observe first)");
    CUDA_TRY(c, cudaEventSynchronize(c->ev_obs_done));
    c->obs_pending = false;
    if (step) *step = c->obs_step;
    const unsigned long long flag = *c->h_obs_flag;
    if (flag != ~0ull) {
        c->latched = true;
        return fail(c, ENS_E_DIVERGED, "non-finite displacement at step " + std::to_string(flag >> 24) +
                                           " in realisation " + std::to_string(flag & 0xffffff));
    }
    return ENS_OK;
}

// N2 (ens_options.persistent): the per-part arguments of the persistent kernel, rebuilt after
// any change that would rebuild the CUDA graphs (traction shape, load table, state)
static int step_persistent(ens_ctx* c, int64_t n) {
    if (!c->d_pparts || c->graph_dirty) {
        std::vector<ens::StepArgs> args;
        std::vector<int64_t> items(1, 0);
        for (Part& p : c->parts) {
            ens::StepArgs a = part_args(c, p);
            a.row0 = 0;
            a.V = p.n_own;
            a.fwd_ptr = p.d_fwd_ptr;
            a.fwd_dst = p.d_fwd_dst;
            a.peer_buf = p.d_peer_buf;
            a.hw_flags = p.d_hflags;          // one part per process: its neighbours' flags
            a.hw_in_q = p.d_in_q;
            a.hw_n_in = p.n_in;
            a.hw_out = p.d_out_flag;
            a.hw_n_out = p.n_out;
            a.hw_err = c->d_herr;
            args.push_back(a);
            items.push_back(items.back() + p.n_own * (c->n_s / ens::pick_vec(c->n_s)));
        }
        dfree(c, c->d_pparts);
        dfree(c, c->d_pitems);
        RC_TRY(upload(c, &c->d_pparts, args.data(), args.size()));
        RC_TRY(upload(c, &c->d_pitems, items.data(), items.size()));
        if (!c->d_pbar) {
            RC_TRY(dalloc(c, &c->d_pbar, 2));
            CUDA_TRY(c, cudaMemsetAsync(c->d_pbar, 0, 2 * sizeof(unsigned int), c->stream));
        }
        c->graph_dirty = false;
    }
    CUDA_TRY(c, ens::launch_steps_persistent(c->d_pparts, c->d_pitems, int32_t(c->parts.size()), c->n_s,
                                             c->kernel == ENS_KERNEL_ASSEMBLED_SYM, n, c->d_pbar, c->multi ? 1 : 0,
                                             c->stream));
    CUDA_TRY(c, ens::launch_advance(c->d_step, n, c->stream));
    c->step += n;
    return ENS_OK;
}

int ens_step(ens_ctx* c, int64_t n) {
    if (!c) return fail(nullptr, ENS_E_ARG, "ctx is NULL");
    if (n < 0) return fail(c, ENS_E_ARG, "n must be >= 0");
    if (c->latched) return fail(c, ENS_E_STATE, "context diverged: call ens_set_state before stepping again");
    if (!c->p2p_connected) return fail(c, ENS_E_STATE, "P2P halo: call ens_p2p_connect before ens_step");
    if (n > 0 && c->coef_dirty) {
        CUDA_TRY(c, ens::launch_seed_coeffs(part_args(c, c->parts[0]), c->stream));
        c->coef_dirty = false;
    }
    if (c->persistent && n > 0) return step_persistent(c, n);
    int64_t left = n;
    if (c->use_graphs() && n >= c->graph_steps) {
        if (c->graph_dirty) drop_graph(c);
        c->graph_dirty = false;
        for (; left >= c->graph_steps; left -= c->graph_steps) {
            const int par = int(c->step & 1);
            if (!c->graph[par]) {
                const int rc = build_graph(c, par);
                if (rc && c->nccl_comm) {
                    // an NCCL build that cannot capture its send/recv: every rank runs the same
                    // code and fails the same way, so all fall back to direct launches together
                    (void)cudaGetLastError();
                    drop_graph(c);
                    c->graph_dirty = false;
                    c->graph_steps = 0;
                    break;
                }
                RC_TRY(rc);
            }
            CUDA_TRY(c, cudaGraphLaunch(c->graph[par], c->stream));
            c->step += c->graph_steps;
        }
    }
    for (int64_t k = 0; k < left; ++k) RC_TRY(enqueue_step(c, c->step, k, c->stream));
    if (left) CUDA_TRY(c, ens::launch_advance(c->d_step, left, c->stream));
    c->step += left;
    return ENS_OK;
}

int ens_prepare(ens_ctx* c) {
    if (!c) return fail(nullptr, ENS_E_ARG, "ctx is NULL");
    if (!c->p2p_connected) return fail(c, ENS_E_STATE, "P2P halo: call ens_p2p_connect before ens_prepare");
    if (!c->use_graphs() || c->persistent) return ENS_OK;
    if (c->graph_dirty) drop_graph(c);
    c->graph_dirty = false;
    for (int par = 0; par < 2; ++par) {
        if (c->graph[par]) continue;
        const int rc = build_graph(c, par);
        if (rc && c->nccl_comm) {          // the same fallback as ens_step (every rank alike)
            (void)cudaGetLastError();
            drop_graph(c);
            c->graph_steps = 0;
            return ENS_OK;
        }
        RC_TRY(rc);
    }
    return ENS_OK;
}

int ens_sync(ens_ctx* c) {
    if (!c) return fail(nullptr, ENS_E_ARG, "ctx is NULL");
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->comm_stream) CUDA_TRY(c, cudaStreamSynchronize(c->comm_stream));
    unsigned long long flag = 0, herr = ~0ull;
    CUDA_TRY(c, cudaMemcpy(&herr, c->d_herr, sizeof(herr), cudaMemcpyDeviceToHost));
    if (herr != ~0ull) {
        c->latched = true;
        return fail(c, ENS_E_CUDA, "P2P halo: step " + std::to_string(herr >> 16) + " waited > 10 s for rank " +
                                       std::to_string(herr & 0xffff));
    }
    CUDA_TRY(c, cudaMemcpy(&flag, c->d_flag, sizeof(flag), cudaMemcpyDeviceToHost));
    if (flag != ~0ull) {
        c->latched = true;
        return fail(c, ENS_E_DIVERGED, "non-finite displacement at step " + std::to_string(flag >> 24) +
                                           " in realisation " + std::to_string(flag & 0xffffff));
    }
    return ENS_OK;
}

static int64_t abi_rows(const ens_ctx* c) { return c->multi ? c->parts[0].n_own : c->V; }

int ens_get_state(ens_ctx* c, double* u_n, double* u_nm1, double* t, int64_t* step) {
    if (!c) return fail(nullptr, ENS_E_ARG, "ctx is NULL");
    const int rc = ens_sync(c);
    if (rc && rc != ENS_E_DIVERGED) return rc;
    const int64_t Vabi = abi_rows(c);
    const size_t n = size_t(Vabi) * 3 * size_t(c->n_s);
    double* outs[2] = {u_n, u_nm1};
    for (int k = 0; k < 2; ++k) {
        if (!outs[k]) continue;
        for (Part& p : c->parts) {
            double* src = ((c->step + k) & 1) ? p.d_u1 : p.d_u0;     // u_n = buf[step & 1]
            CUDA_TRY(c, ens::launch_dev_to_abi(p.n_own, c->n_s, p.d_map_abi, Vabi, src, c->d_stage, c->stream));
        }
        CUDA_TRY(c, cudaMemcpyAsync(outs[k], c->d_stage, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    }
    if (t) *t = double(c->step) * c->dt;
    if (step) *step = c->step;
    return rc;
}

int ens_get_owned(const ens_ctx* c, int32_t* node_ids, int64_t* n) {
    if (!c || !n) return fail(nullptr, ENS_E_ARG, "NULL argument");
    *n = abi_rows(c);
    if (node_ids) {
        if (c->multi) std::copy(c->parts[0].map_own.begin(), c->parts[0].map_own.end(), node_ids);
        else
            for (int64_t i = 0; i < c->V; ++i) node_ids[i] = int32_t(i);
    }
    return ENS_OK;
}

int ens_set_state(ens_ctx* c, const double* u_n, const double* u_nm1, double t, int64_t step) {
    if (!c) return fail(nullptr, ENS_E_ARG, "ctx is NULL");
    if (step < 0) return fail(c, ENS_E_ARG, "step must be >= 0");
    (void)t;   // t = step * dt by construction
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->comm_stream) CUDA_TRY(c, cudaStreamSynchronize(c->comm_stream));
    const size_t n = size_t(c->V) * 3 * size_t(c->n_s);
    const double* ins[2] = {u_n, u_nm1};
    for (int k = 0; k < 2; ++k) {
        if (ins[k]) CUDA_TRY(c, cudaMemcpyAsync(c->d_stage, ins[k], n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
        for (Part& p : c->parts) {
            double* dst = ((step + k) & 1) ? p.d_u1 : p.d_u0;
            const int64_t rows = p.n_own + p.n_gh;
            if (!ins[k]) CUDA_TRY(c, cudaMemsetAsync(dst, 0, size_t(rows) * 3 * size_t(c->n_s) * sizeof(double), c->stream));
            else CUDA_TRY(c, ens::launch_abi_to_dev(rows, c->n_s, p.d_map_all, c->V, c->d_stage, dst, c->stream));
        }
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    }
    static thread_local int64_t h_step;
    h_step = step;
    CUDA_TRY(c, cudaMemcpyAsync(c->d_step, &h_step, sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    CUDA_TRY(c, cudaMemsetAsync(c->d_flag, 0xff, sizeof(unsigned long long), c->stream));
    if (c->p2p()) {      // every ghost row now holds u_step: the neighbours' flags restart at step
        static thread_local std::vector<unsigned long long> h_flags;
        h_flags.assign(size_t(c->world), (unsigned long long)step);
        for (Part& p : c->parts)
            CUDA_TRY(c, cudaMemcpyAsync(p.d_hflags, h_flags.data(), h_flags.size() * sizeof(unsigned long long),
                                        cudaMemcpyHostToDevice, c->stream));
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    c->step = step;
    c->latched = false;
    c->coef_dirty = true;
    return ENS_OK;
}

int ens_apply_stiffness(ens_ctx* c, const double* u, double* y) {
    if (!c || !u || !y) return fail(c, ENS_E_ARG, "ens_apply_stiffness: NULL argument");
    const size_t nfull = size_t(c->V) * 3 * size_t(c->n_s);
    CUDA_TRY(c, cudaMemcpyAsync(c->d_stage, u, nfull * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    for (Part& p : c->parts) {
        const int64_t rows = p.n_own + p.n_gh;
        if (!p.d_scratch_u) {
            RC_TRY(dalloc(c, &p.d_scratch_u, size_t(rows) * 3 * size_t(c->n_s)));
            RC_TRY(dalloc(c, &p.d_scratch_y, size_t(p.n_own) * 3 * size_t(c->n_s)));
        }
        CUDA_TRY(c, ens::launch_abi_to_dev(rows, c->n_s, p.d_map_all, c->V, c->d_stage, p.d_scratch_u, c->stream));
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    const int64_t Vabi = abi_rows(c);
    for (Part& p : c->parts) {
        ens::StepArgs a = part_args(c, p);
        a.ubuf0 = a.ubuf1 = p.d_scratch_u;
        a.y_out = p.d_scratch_y;
        CUDA_TRY(c, launch_rows(c, p, a, 0, p.n_own, c->stream));
        CUDA_TRY(c, ens::launch_dev_to_abi(p.n_own, c->n_s, p.d_map_abi, Vabi, p.d_scratch_y, c->d_stage, c->stream));
    }
    CUDA_TRY(c, cudaMemcpyAsync(y, c->d_stage, size_t(Vabi) * 3 * size_t(c->n_s) * sizeof(double),
                                cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return ENS_OK;
}

static int observe_check(ens_ctx* c) {
    if (c->parts.size() != 1 || c->multi || c->h_tris.empty())
        return fail(c, ENS_E_UNSUPPORTED, "stresses / statistics need a single-part context created by ens_create");
    return ENS_OK;
}

int ens_stress(ens_ctx* c, int32_t frame, const double* centerline, int32_t n_c, double* sigma, double* mean,
               double* q05, double* q95) {
    if (!c) return fail(nullptr, ENS_E_ARG, "ctx is NULL");
    if (frame < 0 || frame > 1) return fail(c, ENS_E_ARG, "frame must be 0 (local) or 1 (centreline)");
    if (centerline && n_c < 2) return fail(c, ENS_E_ARG, "centerline needs n_c >= 2 points");
    RC_TRY(observe_check(c));
    const int rc = ens_sync(c);
    if (rc && rc != ENS_E_DIVERGED) return rc;
    const int64_t F = c->F, n_s = c->n_s;
    if (!c->d_G) {
        std::vector<double> Gh(size_t(F) * 45), R(9);
        std::vector<int32_t> et(size_t(F) * 3);
        for (int64_t e = 0; e < F; ++e) {
            const int32_t* t = c->h_tris.data() + 3 * e;
            ens::element_strain_operator(&c->h_xyz[3 * size_t(t[0])], &c->h_xyz[3 * size_t(t[1])],
                                         &c->h_xyz[3 * size_t(t[2])], Gh.data() + 45 * e, R.data());
            for (int a = 0; a < 3; ++a) et[size_t(3 * e + a)] = c->iperm[size_t(t[a])];
        }
        RC_TRY(upload(c, &c->d_G, Gh.data(), Gh.size()));
        RC_TRY(upload(c, &c->d_etri, et.data(), et.size()));
    }
    std::vector<double> Mh(size_t(F) * 9), Gtmp(45), R(9);
    for (int64_t e = 0; e < F; ++e) {
        const int32_t* t = c->h_tris.data() + 3 * e;
        const double* X[3] = {&c->h_xyz[3 * size_t(t[0])], &c->h_xyz[3 * size_t(t[1])], &c->h_xyz[3 * size_t(t[2])]};
        ens::element_strain_operator(X[0], X[1], X[2], Gtmp.data(), R.data());
        const double cen[3] = {(X[0][0] + X[1][0] + X[2][0]) / 3.0, (X[0][1] + X[1][1] + X[2][1]) / 3.0,
                               (X[0][2] + X[1][2] + X[2][2]) / 3.0};
        ens::stress_frame(cen, R.data(), frame, centerline, n_c, Mh.data() + 9 * e);
    }
    double *d_M = nullptr, *d_out = nullptr;
    RC_TRY(upload(c, &d_M, Mh.data(), Mh.size()));
    RC_TRY(dalloc(c, &d_out, size_t(F) * 6 * size_t(n_s)));
    const Part& p = c->parts[0];
    const double* un = (c->step & 1) ? p.d_u1 : p.d_u0;
    CUDA_TRY(c, ens::launch_stress(F, c->n_s, frame, c->d_etri, c->d_G, d_M, c->d_Ebar, c->nu, c->k_shear, un, d_out,
                                   c->stream));
    if (sigma) {
        double* d_abi = nullptr;
        RC_TRY(dalloc(c, &d_abi, size_t(F) * 6 * size_t(n_s)));
        CUDA_TRY(c, ens::launch_to_abi(F, 6, c->n_s, nullptr, d_out, d_abi, c->stream));
        CUDA_TRY(c, cudaMemcpyAsync(sigma, d_abi, size_t(F) * 6 * size_t(n_s) * sizeof(double), cudaMemcpyDeviceToHost,
                                    c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        dfree(c, d_abi);
    }
    if (mean || q05 || q95) {
        const int64_t n_seg = F * 6;
        double *d_sorted = nullptr, *d_st = nullptr;
        unsigned char* d_tmp = nullptr;
        const size_t tb = ens::stats_temp_bytes(n_seg, c->n_s);
        RC_TRY(dalloc(c, &d_sorted, size_t(n_seg) * size_t(n_s)));
        RC_TRY(dalloc(c, &d_tmp, tb));
        RC_TRY(dalloc(c, &d_st, size_t(n_seg) * 3));
        CUDA_TRY(c, ens::ensemble_stats(n_seg, c->n_s, 6, nullptr, 6, 0, d_out, d_sorted, d_tmp, tb, d_st, d_st + n_seg,
                                        d_st + 2 * n_seg, c->stream));
        double* outs[3] = {mean, q05, q95};
        for (int k = 0; k < 3; ++k)
            if (outs[k])
                CUDA_TRY(c, cudaMemcpyAsync(outs[k], d_st + k * n_seg, size_t(n_seg) * sizeof(double),
                                            cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        dfree(c, d_sorted);
        dfree(c, d_tmp);
        dfree(c, d_st);
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    dfree(c, d_M);
    dfree(c, d_out);
    return rc;
}

int ens_displacement_stats(ens_ctx* c, double* mean, double* q05, double* q95) {
    if (!c) return fail(nullptr, ENS_E_ARG, "ctx is NULL");
    RC_TRY(observe_check(c));
    const int rc = ens_sync(c);
    if (rc && rc != ENS_E_DIVERGED) return rc;
    const int64_t V = c->V, n_s = c->n_s;
    const Part& p = c->parts[0];
    const double* un = (c->step & 1) ? p.d_u1 : p.d_u0;
    double *d_mag = nullptr, *d_sorted = nullptr, *d_st = nullptr;
    unsigned char* d_tmp = nullptr;
    const size_t tb = ens::stats_temp_bytes(3 * V, c->n_s);
    RC_TRY(dalloc(c, &d_mag, size_t(V) * size_t(n_s)));
    RC_TRY(dalloc(c, &d_sorted, size_t(3 * V) * size_t(n_s)));
    RC_TRY(dalloc(c, &d_tmp, tb));
    RC_TRY(dalloc(c, &d_st, size_t(V) * 4 * 3));
    CUDA_TRY(c, ens::launch_magnitude(V, c->n_s, un, d_mag, c->stream));
    // components: segments (row i, c) of u itself; rows written at the caller's node id
    CUDA_TRY(c, ens::ensemble_stats(3 * V, c->n_s, 3, p.d_map_own, 4, 0, un, d_sorted, d_tmp, tb, d_st, d_st + 4 * V,
                                    d_st + 8 * V, c->stream));
    CUDA_TRY(c, ens::ensemble_stats(V, c->n_s, 1, p.d_map_own, 4, 3, d_mag, d_sorted, d_tmp, tb, d_st, d_st + 4 * V,
                                    d_st + 8 * V, c->stream));
    double* outs[3] = {mean, q05, q95};
    for (int k = 0; k < 3; ++k)
        if (outs[k])
            CUDA_TRY(c, cudaMemcpyAsync(outs[k], d_st + k * 4 * V, size_t(V) * 4 * sizeof(double), cudaMemcpyDeviceToHost,
                                        c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    dfree(c, d_mag);
    dfree(c, d_sorted);
    dfree(c, d_tmp);
    dfree(c, d_st);
    return rc;
}

int ens_matern_fields(const ens_mesh* mesh, double rho_corr, int32_t n, const double* z, double* x, double tol,
                      int32_t max_iter, const ens_options* opt, int32_t* iters, double* max_rel_res) {
    if (!mesh || !z || !x || n < 1) return fail(nullptr, ENS_E_ARG, "ens_matern_fields: bad arguments");
    if (!(rho_corr > 0.0) || !std::isfinite(rho_corr)) return fail(nullptr, ENS_E_ARG, "rho_corr must be > 0");
    if (!(tol > 0.0) || max_iter < 1) return fail(nullptr, ENS_E_ARG, "tol must be > 0 and max_iter >= 1");
    if (mesh->n_nodes < 1 || mesh->n_tris < 1 || !mesh->xyz || !mesh->tris)
        return fail(nullptr, ENS_E_ARG, "mesh needs nodes and triangles");
    ens::MeshView m{mesh->n_nodes, mesh->n_tris, mesh->xyz, mesh->tris};
    int64_t bad = -1;
    if (ens::validate_mesh(m, &bad)) return fail(nullptr, ENS_E_MESH, "invalid mesh (element / node " + std::to_string(bad) + ")");
    ens_ctx tmp;               // allocation plumbing only
    ens_ctx* c = &tmp;
    auto body = [&]() -> int {
        RC_TRY(init_ctx(c, opt));
        const int64_t V = m.V;
        const ens::Pattern pat = ens::build_pattern(m);
        const double kappa = std::sqrt(8.0) / rho_corr;                 // PAPER.md:67, nu = 1
        std::vector<double> val, diag, lumped;
        ens::gmrf_system(m, pat, kappa, val, diag, lumped);
        std::vector<double> dinv(static_cast<size_t>(V)), sq(static_cast<size_t>(V));
        for (int64_t i = 0; i < V; ++i) {
            dinv[size_t(i)] = 1.0 / diag[size_t(i)];
            sq[size_t(i)] = std::sqrt(lumped[size_t(i)]);
        }
        std::vector<int32_t> rp(pat.row_ptr.begin(), pat.row_ptr.end());
        ens::GmrfSystem S;
        S.V = V;
        int32_t *d_rp, *d_col, *d_perm;
        double *d_val, *d_dinv, *d_sq, *d_z, *d_x, *d_w;
        RC_TRY(upload(c, &d_rp, rp.data(), rp.size()));
        RC_TRY(upload(c, &d_col, pat.col.data(), pat.col.size()));
        RC_TRY(upload(c, &d_perm, pat.perm.data(), pat.perm.size()));
        RC_TRY(upload(c, &d_val, val.data(), val.size()));
        RC_TRY(upload(c, &d_dinv, dinv.data(), dinv.size()));
        RC_TRY(upload(c, &d_sq, sq.data(), sq.size()));
        RC_TRY(upload(c, &d_z, z, size_t(V) * size_t(n)));
        RC_TRY(dalloc(c, &d_x, size_t(V) * size_t(n)));
        RC_TRY(dalloc(c, &d_w, ens::gmrf_work_doubles(V, n)));
        S.rp = d_rp;
        S.col = d_col;
        S.val = d_val;
        S.dinv = d_dinv;
        S.sqrtC = d_sq;
        S.perm = d_perm;
        // unit marginal variance: sigma^2 = Gamma(nu) / (Gamma(nu + d/2) (4 pi)^{d/2} kappa^{2 nu})
        // = 1 / (4 pi kappa^2) for nu = 1, d = 2
        const double scale = 1.0 / std::sqrt(1.0 / (4.0 * M_PI * kappa * kappa));
        CUDA_TRY(c, ens::gmrf_pcg(S, n, d_z, d_x, scale, tol, max_iter, d_w, c->stream, iters, max_rel_res));
        CUDA_TRY(c, cudaMemcpyAsync(x, d_x, size_t(V) * size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
        return ENS_OK;
    };
    const int rc = body();
    free_all(c);
    return rc;
}

// ---- P2P halo across processes (CUDA IPC) -------------------------------------------------
namespace {
struct P2PBlob {
    uint32_t magic;
    int32_t rank, world, n_s;
    int64_t n_loc;
    cudaIpcMemHandle_t u0, u1, flags;
};
static_assert(sizeof(P2PBlob) <= ENS_P2P_BLOB_BYTES, "blob");
constexpr uint32_t kBlobMagic = 0x32503245u;
}  // namespace

int ens_p2p_export(const ens_ctx* c, void* blob) {
    if (!c || !blob) return fail(nullptr, ENS_E_ARG, "NULL argument");
    ens_ctx* m = const_cast<ens_ctx*>(c);
    if (!(c->multi && c->p2p())) return fail(m, ENS_E_STATE, "not a one-part-per-process P2P context");
    const Part& p = c->parts[0];
    P2PBlob b{};
    b.magic = kBlobMagic;
    b.rank = c->rank;
    b.world = c->world;
    b.n_s = c->n_s;
    b.n_loc = p.n_own + p.n_gh;
    CUDA_TRY(m, cudaIpcGetMemHandle(&b.u0, p.d_u0));
    CUDA_TRY(m, cudaIpcGetMemHandle(&b.u1, p.d_u1));
    CUDA_TRY(m, cudaIpcGetMemHandle(&b.flags, p.d_hflags));
    std::memset(blob, 0, ENS_P2P_BLOB_BYTES);
    std::memcpy(blob, &b, sizeof(b));
    return ENS_OK;
}

int ens_p2p_connect(ens_ctx* c, const void* blobs) {
    if (!c || !blobs) return fail(nullptr, ENS_E_ARG, "NULL argument");
    if (!(c->multi && c->p2p())) return fail(c, ENS_E_STATE, "not a one-part-per-process P2P context");
    if (c->p2p_connected) return fail(c, ENS_E_STATE, "already connected");
    Part& P = c->parts[0];
    std::vector<double*> pb;
    std::vector<unsigned long long*> of;
    for (size_t k = 0; k < P.out_q.size(); ++k) {
        const int32_t q = P.out_q[k];
        P2PBlob b;
        std::memcpy(&b, static_cast<const char*>(blobs) + size_t(q) * ENS_P2P_BLOB_BYTES, sizeof(b));
        if (b.magic != kBlobMagic || b.rank != q || b.world != c->world || b.n_s != c->n_s || b.n_loc != P.out_rows[k])
            return fail(c, ENS_E_ARG, "P2P blob of rank " + std::to_string(q) + " does not match this context");
        void* ptr[3] = {nullptr, nullptr, nullptr};
        const cudaIpcMemHandle_t* h[3] = {&b.u0, &b.u1, &b.flags};
        for (int j = 0; j < 3; ++j) {
            CUDA_TRY(c, cudaIpcOpenMemHandle(&ptr[j], *h[j], cudaIpcMemLazyEnablePeerAccess));
            c->ipc_opened.push_back(ptr[j]);
        }
        pb.push_back(static_cast<double*>(ptr[0]));
        pb.push_back(static_cast<double*>(ptr[1]));
        of.push_back(static_cast<unsigned long long*>(ptr[2]) + P.plan.p);
    }
    if (!pb.empty()) {
        CUDA_TRY(c, cudaMemcpyAsync(P.d_peer_buf, pb.data(), pb.size() * sizeof(double*), cudaMemcpyHostToDevice,
                                    c->stream));
        CUDA_TRY(c, cudaMemcpyAsync(P.d_out_flag, of.data(), of.size() * sizeof(void*), cudaMemcpyHostToDevice,
                                    c->stream));
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    c->p2p_connected = true;
    return ENS_OK;
}

int ens_measure_fp64(int32_t device, double* tflops) {
    if (!tflops) return fail(nullptr, ENS_E_ARG, "tflops is NULL");
    if (device >= 0) {
        cudaError_t e = cudaSetDevice(device);
        if (e != cudaSuccess) return cuda_fail(nullptr, e, "cudaSetDevice");
    }
    cudaError_t e = ens::measure_fp64_fma(tflops);
    if (e != cudaSuccess) return cuda_fail(nullptr, e, "fp64 FMA probe");
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
    info->graph_steps = (c->use_graphs() && !c->persistent) ? c->graph_steps : 0;
    info->reassemble_every = c->reassemble_every;
    info->halo = c->halo;
    info->mf_variant = c->kernel == ENS_KERNEL_MATRIX_FREE ? c->mf_variant : 0;
    info->mfs_consumers = info->mfs_unit_width = info->mfs_stage_width = info->mfs_stages = 0;
    if (c->kernel == ENS_KERNEL_MATRIX_FREE && c->mf_variant == ENS_MF_STAGED) {
        const ens::MfsShape sh = ens::mf_staged_shape(c->mfs_plan.shape);
        info->mfs_consumers = sh.consumers;
        info->mfs_unit_width = 64 * c->mfs_plan.ws;
        info->mfs_stage_width = ens::mfs_stage_w(c->mfs_plan, c->n_s);
        info->mfs_stages = sh.stages;
    }
    info->comm_rank = info->comm_nranks = -1;
    if (c->nccl_comm && c->nccl && c->nccl->comm_count && c->nccl->comm_user_rank) {
        int r = -1, n = -1;
        if (c->nccl->comm_user_rank(c->nccl_comm, &r) == 0 && c->nccl->comm_count(c->nccl_comm, &n) == 0) {
            info->comm_rank = r;
            info->comm_nranks = n;
        }
    }
    // algorithmic HBM bytes of the rows this context advances: values +
    // u_n, u_{n-1} read, u_{n+1} written, c1 (+ c2, c3) per node per realisation
    const int64_t ns = c->n_s, per_node = 3 * 8 * 3 + 8 + (c->damping == ENS_DAMP_IDENTITY ? 16 : 0);
    int64_t own = 0, halo = 0, launches = 0;
    for (const Part& p : c->parts) {
        own += p.n_own;
        halo += int64_t(p.plan.send_rows.size());
        for (const auto& pe : p.plan.peers) halo += pe.recv_n;
        if (!c->has_halo()) launches += 1;
        else if (c->persistent) launches = 1;             // one launch per ens_step call
        else if (c->p2p() && halo_fused(c) && (p.plan.b_lo > 0 || p.plan.b_hi > 0))
            launches += 1 + (p.plan.b_lo > 0) + (p.plan.b_hi > 0);
        else if (c->p2p()) launches += 1 + (p.n_in > 0) + (p.plan.b_lo > 0) + (p.plan.b_hi > 0) + (p.n_out > 0);
        else launches += 1 + (p.plan.b_lo > 0) + (p.plan.b_hi > 0) + !p.plan.send_rows.empty();
    }
    info->n_owned = own;
    info->halo_bytes_per_step = halo * 3 * 8 * ns;
    info->launches_per_step = int32_t(launches);
    const double frac = c->V ? double(own) / double(c->V) : 1.0;
    int64_t stored = 0;
    for (const Part& p : c->parts) stored += p.n_stored;
    if (c->kernel == ENS_KERNEL_ASSEMBLED) {
        info->bytes_per_step = int64_t(frac * double(ns * (72 * c->nnzb + per_node * c->V)));
        info->flops_per_step = int64_t(frac * double(ns * (18 * c->nnzb + 3 * 5 * c->V)));
    } else if (c->kernel == ENS_KERNEL_ASSEMBLED_SYM) {
        info->bytes_per_step = ns * (72 * stored + int64_t(frac * double(per_node * c->V)));
        info->flops_per_step = int64_t(frac * double(ns * (18 * c->nnzb + 3 * 5 * c->V)));
    } else {
        // K^: the 2 x 9 (prev, next) values of each of an element's 3 rows = 432 B per element
        // (DIFF), else the full 9 x 9 = 648 B.  Flops per incidence: DIFF 18 FMA + 3 adds + the
        // alpha FMA on 3 components + the 3-component difference of the new neighbour = 48;
        // else 27 FMA + 2 x 3 adds + 3 alpha FMA = 66 (counted 60: the adds folded)
        const bool dif = ens::mf_diff();
        info->bytes_per_step = int64_t(frac * double(ns * (8 * c->F + per_node * c->V) + (dif ? 432 : 648) * c->F));
        info->flops_per_step = int64_t(frac * double(ns * (3 * c->F * (dif ? 48 : 60) + 3 * 5 * c->V)));
    }
    return ENS_OK;
}

void ens_destroy(ens_ctx* c) {
    if (!c) return;
    free_all(c);
    delete c;
}

const char* ens_last_error(const ens_ctx* c) { return c ? c->err.c_str() : g_err.c_str(); }

// ---- host-side maps ------------------------------------------------------------------

int ens_host_validate(int64_t n_nodes, int64_t n_tris, const double* xyz, const int32_t* tris, int32_t* code,
                      int64_t* bad) {
    ens::MeshView m{n_nodes, n_tris, xyz, tris};
    int64_t b = -1;
    const int v = ens::validate_mesh(m, &b);
    if (code) *code = v;
    if (bad) *bad = b;
    return v ? ENS_E_MESH : ENS_OK;
}

int ens_host_pattern(int64_t n_nodes, int64_t n_tris, const int32_t* tris, int32_t* perm, int64_t* row_ptr,
                     int32_t* col, int64_t col_cap, int64_t* nnzb) {
    ens::MeshView m{n_nodes, n_tris, nullptr, tris};
    const ens::Pattern p = ens::build_pattern(m);
    *nnzb = int64_t(p.col.size());
    if (*nnzb > col_cap) return fail(nullptr, ENS_E_ARG, "col_cap too small");
    std::copy(p.perm.begin(), p.perm.end(), perm);
    std::copy(p.row_ptr.begin(), p.row_ptr.end(), row_ptr);
    std::copy(p.col.begin(), p.col.end(), col);
    return ENS_OK;
}

int ens_host_partition(int64_t n_nodes, const int64_t* row_ptr, int32_t n_parts, int64_t* bounds) {
    if (n_parts < 1) return fail(nullptr, ENS_E_ARG, "n_parts must be >= 1");
    const std::vector<int64_t> rp(row_ptr, row_ptr + n_nodes + 1);
    const auto b = ens::partition_bounds(rp, n_parts);
    std::copy(b.begin(), b.end(), bounds);
    return ENS_OK;
}

int ens_host_ghosts(int64_t n_nodes, const int64_t* row_ptr, const int32_t* col, int64_t lo, int64_t hi,
                    int32_t* ghosts, int64_t cap, int64_t* n) {
    const std::vector<int64_t> rp(row_ptr, row_ptr + n_nodes + 1);
    const std::vector<int32_t> cl(col, col + row_ptr[n_nodes]);
    const auto g = ens::ghost_rows(rp, cl, lo, hi);
    *n = int64_t(g.size());
    if (*n > cap) return fail(nullptr, ENS_E_ARG, "cap too small");
    std::copy(g.begin(), g.end(), ghosts);
    return ENS_OK;
}

int ens_host_halo_plan(int64_t n_nodes, const int64_t* row_ptr, const int32_t* col, int32_t n_parts, int32_t part,
                       int64_t* lo_hi_b, int32_t* peers, int64_t* peer_info, int32_t* send_rows, int64_t cap,
                       int64_t* n_peers, int64_t* n_send) {
    if (n_parts < 1 || part < 0 || part >= n_parts) return fail(nullptr, ENS_E_ARG, "bad part");
    const std::vector<int64_t> rp(row_ptr, row_ptr + n_nodes + 1);
    const std::vector<int32_t> cl(col, col + row_ptr[n_nodes]);
    const auto plans = ens::halo_plan(rp, cl, n_parts);
    const auto& pl = plans[size_t(part)];
    *n_peers = int64_t(pl.peers.size());
    *n_send = int64_t(pl.send_rows.size());
    if (*n_peers > n_parts || *n_send > cap) return fail(nullptr, ENS_E_ARG, "cap too small");
    lo_hi_b[0] = pl.lo;
    lo_hi_b[1] = pl.hi;
    lo_hi_b[2] = pl.b_lo;
    lo_hi_b[3] = pl.b_hi;
    lo_hi_b[4] = int64_t(pl.ghosts.size());
    for (size_t k = 0; k < pl.peers.size(); ++k) {
        peers[k] = pl.peers[k].q;
        peer_info[4 * k + 0] = pl.peers[k].send_off;
        peer_info[4 * k + 1] = pl.peers[k].send_n;
        peer_info[4 * k + 2] = pl.peers[k].recv_row;
        peer_info[4 * k + 3] = pl.peers[k].recv_n;
    }
    std::copy(pl.send_rows.begin(), pl.send_rows.end(), send_rows);
    return ENS_OK;
}

int ens_host_mf_tiles(int64_t n_nodes, int64_t n_tris, const double* xyz, const int32_t* tris, int32_t n_s,
                      int32_t patches, int32_t max_rows, int64_t stage_bytes, int32_t* tile_of,
                      int64_t* tile_bytes, int32_t* tile_entries, int64_t* n_tiles, int64_t* budget) {
    if (n_s < 64 || n_s % 64 || max_rows < 1 || max_rows > ens::kMfsMaxRows)
        return fail(nullptr, ENS_E_ARG, "ens_host_mf_tiles: n_s % 64 == 0 and 1 <= max_rows <= 32");
    ens::MeshView m{n_nodes, n_tris, xyz, tris};
    int64_t bad = -1;
    if (ens::validate_mesh(m, &bad)) return fail(nullptr, ENS_E_MESH, "invalid mesh");
    const ens::Pattern pat = ens::build_pattern(m);
    std::vector<double> Khat(size_t(81 * n_tris)), area(static_cast<size_t>(n_tris));
    for (int64_t e = 0; e < n_tris; ++e)
        ens::element_stiffness(xyz + 3 * int64_t(tris[3 * e]), xyz + 3 * int64_t(tris[3 * e + 1]),
                               xyz + 3 * int64_t(tris[3 * e + 2]), 0.5, 5.0 / 6.0, Khat.data() + 81 * e, area.data() + e);
    const ens::Fans fans = ens::build_fans(m, pat.iperm, Khat);
    ens::MfsPlan plan = ens::mf_staged_plan(n_s);
    plan.patches = patches != 0;
    plan.max_rows = max_rows;
    const size_t SB = stage_bytes > 0 ? size_t(stage_bytes) : size_t(ens::mf_staged_shape(plan.shape).stage_bytes);
    const size_t US = size_t(n_s) * 24, AS = size_t(n_s) * 8;
    // element ids as build_part numbers them for the matrix-free kernels (first touch)
    std::vector<ens::FanRec> rec = fans.rec;
    std::vector<int32_t> first(static_cast<size_t>(n_tris), -1);
    int32_t next = 0;
    for (auto& r : rec) {
        if (first[size_t(r.e)] < 0) first[size_t(r.e)] = next++;
        r.e = first[size_t(r.e)];
    }
    const auto tiles = mf_patches(fans.ptr, rec, n_nodes, 0, n_nodes, US, AS, SB, plan);
    MfLayout L;
    for (size_t t = 0; t < tiles.size(); ++t) {
        for (int32_t r : tiles[t]) tile_of[size_t(r)] = int32_t(t);
        mf_layout(fans.ptr, rec, tiles[t], US, AS, L);
        tile_bytes[t] = int64_t(L.bytes);
        tile_entries[t] = L.entries;
    }
    *n_tiles = int64_t(tiles.size());
    *budget = int64_t(SB);
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
