/*
 * ens.h -- C ABI of the B200-native ensemble explicit shell solver (arXiv 2101.09059).
 *
 * The hot path is one explicit central-difference step of N_s wall realisations at once
 * (PAPER.md = the paper's LaTeX source):
 *
 *   (M~ + dt/2 C~) u_{n+1} = dt^2 f_n - (dt^2 K - 2M) u_n - (M - dt/2 C) u_{n-1}
 *                                                (Eq. 22)
 *
 * with K = K(theta_s) the 3-dof linear membrane + transverse-shear shell stiffness of
 * realisation s (Eqs. 7-10), M~ the lumped diagonal mass and C~ the
 * diagonal damping, f_n the prescribed wall traction of the one-way
 * coupled fluid solve, applied to all realisations at once ("solving
 * multiple realizations ... at the same time"; "no approximation
 * introduced").  The product K_s u_s is an ensemble sparse
 * matrix-multi-vector product on one shared block-CSR pattern with 9 N_s values per
 * block ("dense coefficient entries of size 9 n_s") or its matrix-free
 * element form scaled by E*zeta at the Gauss points.
 *
 * Conventions (all calls)
 *   - Units CGS: cm, g, s, Ba = dyn/cm^2.
 *   - Host arrays passed IN are read during the call and never retained: the library
 *     copies everything it needs before returning (ownership stays with the caller).
 *   - Ensemble arrays crossing the ABI are realisation-OUTERMOST in the caller's node
 *     numbering: u[n_s][n_nodes][3], E[n_s][n_nodes], h[n_s][n_nodes].  Inside, the
 *     device layout is realisation-innermost in RCM order.
 *   - Return value: ENS_OK (0) or a negative ENS_E_* code; ens_last_error() gives a
 *     message naming the offending argument / element / edge / step.
 *   - A context is not thread-safe; distinct contexts are independent.
 *   - Device memory is owned by the context, obtained through opt->dev_alloc (the
 *     PyTorch caching allocator in the Python binding) or cudaMallocAsync if NULL.
 *   - Every floating-point quantity is IEEE fp64.
 */
#ifndef ENS_H_
#define ENS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ENS_ABI_VERSION 2

enum {
    ENS_OK = 0,
    ENS_E_ARG = -1,         /* invalid argument (n_s < 1, E <= 0, h <= 0, rho <= 0, nu not in [0, 0.5], bad dt ...) */
    ENS_E_MESH = -2,        /* invalid mesh: node index out of range, repeated node, degenerate triangle,
                               edge shared by > 2 triangles */
    ENS_E_OOM = -3,         /* device allocation failed */
    ENS_E_CUDA = -4,        /* CUDA runtime error (no device, launch failure, ...) */
    ENS_E_NCCL = -5,        /* NCCL error (node-partitioned mode) */
    ENS_E_DIVERGED = -6,    /* a non-finite displacement appeared (step and realisation in the message) */
    ENS_E_STATE = -7,       /* context latched after divergence: call ens_set_state first */
    ENS_E_UNSUPPORTED = -8  /* option combination not built */
};

/* Bits of ens_mesh.fixed[i]: bit c set => displacement component c (x, y, z) of node i is
 * held at zero (fully fixed ends: value 7). */
#define ENS_FIX_X 1
#define ENS_FIX_Y 2
#define ENS_FIX_Z 4

typedef struct {
    int64_t n_nodes;        /* V >= 1 */
    int64_t n_tris;         /* F >= 1 */
    const double* xyz;      /* [V][3] node coordinates, cm */
    const int32_t* tris;    /* [F][3] 0-based node ids, counter-clockwise about the outward normal */
    const uint8_t* fixed;   /* [V] Dirichlet bitmask (ENS_FIX_*), or NULL = none fixed */
} ens_mesh;

typedef struct {
    int32_t n_s;            /* number of realisations held by this context (>= 1) */
    const double* E;        /* [n_s][V] nodal Young's modulus, Ba (> 0)  (Eq. 11) */
    const double* h;        /* [n_s][V] nodal wall thickness zeta, cm (> 0) */
    double rho;             /* wall density, g/cm^3 (> 0); 1.06 */
    double nu;              /* Poisson ratio in [0, 0.5] (Eq. 9; not stated in the paper) */
    double k_shear;         /* transverse shear factor k (> 0), 5/6 */
    int32_t s_begin;        /* global index of realisation 0 of this context (ensemble shards);
                               used only in diagnostics */
} ens_materials;

enum { ENS_DAMP_NONE = 0, ENS_DAMP_MASS = 1, ENS_DAMP_IDENTITY = 2 };
enum { ENS_KERNEL_ASSEMBLED = 0, ENS_KERNEL_MATRIX_FREE = 1, ENS_KERNEL_ASSEMBLED_SYM = 2 };
enum { ENS_DIST_SINGLE = 0, ENS_DIST_NODE = 1, ENS_DIST_ENSEMBLE = 2 };
enum { ENS_HALO_NCCL = 0, ENS_HALO_P2P = 1 };

typedef struct {
    double dt;              /* time step, s; <= 0 => cfl_safety * l_min / sqrt(E_max / rho) */
    double cfl_safety;      /* 0 => 0.9 */
    double c_d;             /* damping coefficient */
    int32_t damping;        /* ENS_DAMP_*: NONE C~ = 0; MASS C~ = c_d M~ (1/s); IDENTITY C~ = c_d I (g/s) */
    int32_t kernel;         /* ENS_KERNEL_*: ASSEMBLED (per-realisation block-CSR values, 9 N_s per block,
                               PAPER.md:349); ASSEMBLED_SYM (the same with only the blocks (i, j >= i)
                               stored: K_s is symmetric, results bit-identical, ~half the bytes);
                               MATRIX_FREE (alpha_{e,s} K^_e per element) */
    int32_t dist;           /* ENS_DIST_*.  ENSEMBLE: this context holds realisations [s_begin, s_begin + n_s)
                               of a sharded ensemble (no communication).  NODE: the RCM rows are split
                               into `world` parts balanced by blocks, each advanced with a halo
                               exchange of the N_s-wide interface rows per step:
                               with nccl_comm != NULL this process holds part `rank` and exchanges with
                               NCCL point-to-point; with nccl_comm == NULL this context holds all
                               `world` parts on one device and exchanges by device copies (single-
                               process emulation; results are bit-identical to ENS_DIST_SINGLE). */
    int32_t rank, world;    /* process-group position (dist == NODE) */
    void* nccl_comm;        /* ncclComm_t of this process group (torch ProcessGroupNCCL._comm_ptr()),
                               resolved against the libnccl.so.2 already loaded in-process */
    void* stream;           /* cudaStream_t all work is enqueued on (NULL = legacy default stream) */
    void* (*dev_alloc)(size_t bytes, void* user);    /* optional device allocator */
    void (*dev_free)(void* ptr, void* user);
    void* alloc_user;
    int32_t device;         /* CUDA device ordinal; < 0 => current device */
    int32_t reassemble_every; /* k > 0: before every step index m >= 1 with m % k == 0 rebuild each
                               realisation's stiffness on its deformed geometry X + u_m (
                               assembled kernels only; mass and loads stay on the reference
                               geometry); 0 = linear, K fixed */
    int32_t halo;           /* dist == NODE: how the interface rows travel (SURVEY.md
                               §8(f) N2).  ENS_HALO_NCCL: boundary rows, send-pack, NCCL send/recv on
                               a comm stream (or device copies when this context holds every part).
                               ENS_HALO_P2P: the boundary-row kernel stores each u_{n+1} send row
                               straight into the neighbours' ghost rows (peer memory over NVLink /
                               the same device), then a one-thread kernel publishes a per-neighbour
                               step counter (st.release.sys) that the neighbour's next step waits for
                               (ld.acquire.sys); no pack, no NCCL, and the step loop is captured in
                               CUDA graphs.  With p2p_procs == 0 this context holds all `world` parts;
                               with p2p_procs == 1 it holds part `rank` and must be connected to the
                               other ranks with ens_p2p_export / ens_p2p_connect before ens_step. */
    int32_t p2p_procs;      /* halo == P2P: 1 = one part per process (CUDA IPC), 0 = all parts here */
    int32_t mf_variant;     /* kernel == MATRIX_FREE: the device data path of the same arithmetic
                               (ENS_MF_*).  AUTO (0): STAGED where it applies (even N_s >= 64), else
                               TILES.  Asking for a path that does not apply to the context
                               (STAGED: N_s odd or < 64; WARP: N_s % 64 != 0 or damping == IDENTITY)
                               returns ENS_E_UNSUPPORTED.  Ignored by the assembled kernels. */
    int32_t persistent;     /* dist == NODE, halo == P2P, kernel ASSEMBLED or ASSEMBLED_SYM, no
                               re-assembly: 1 = ens_step(n) advances every part held here by n
                               steps in ONE persistent cooperative kernel (grid-wide barrier per
                               step, the neighbours' step flags waited for and published inside:
                               SURVEY.md §8(f) N2) instead of CUDA graphs of per-step launches.
                               Other combinations: ENS_E_UNSUPPORTED. */
} ens_options;

/* Matrix-free data paths (ens_options.mf_variant, ens_info.mf_variant).  All three compute
 * the same sums in the same order per row (bit-identical results):
 *   TILES  (1)  k_step_matrix_free: CTA tiles of rows, K^ rows staged by TMA, u and alpha
 *               gathered through L1 into registers; any N_s.
 *   WARP   (2)  k_step_mf_warp: per-warp rings of per-operand TMA copies (item programs).
 *   STAGED (3)  k_step_mf_staged: warp-specialised persistent CTAs; a producer warp stages
 *               whole tiles (the u_n rows of the tile's node set, its alpha rows, records and
 *               K^) by runs of consecutive ids into an mbarrier ring, consumer warps compute
 *               from shared memory. */
enum { ENS_MF_AUTO = 0, ENS_MF_TILES = 1, ENS_MF_WARP = 2, ENS_MF_STAGED = 3 };

typedef struct ens_ctx ens_ctx;

typedef struct {
    double dt, dt_cfl;
    int64_t n_nodes, n_tris, nnzb;      /* nnzb: 3x3 blocks of the pattern (= V + 2 #edges) */
    int32_t n_s, kernel, damping, dist;
    int64_t step;                       /* steps taken since t = 0 (t = step * dt) */
    int64_t bytes_per_step;             /* algorithmic HBM bytes of one fused step */
    int64_t flops_per_step;             /* algorithmic fp64 flops of one fused step */
    int64_t device_bytes;               /* device memory held by the context */
    int32_t rcm_bandwidth;              /* max |i - j| over the pattern in RCM order */
    int64_t n_owned;                    /* rows advanced by this context (V unless NODE with NCCL) */
    int64_t halo_bytes_per_step;        /* bytes sent + received by the halo exchange per step */
    int32_t launches_per_step;          /* kernels per time step (1 without a halo) */
    int32_t reassemble_every;           /* ens_options.reassemble_every */
    int32_t graph_steps;                /* ens_step replays a CUDA graph of this many steps + 1 counter
                                           advance (env ENS_GRAPH_STEPS; 0 = direct launches) */
    int32_t halo;                       /* ens_options.halo (NODE contexts) */
    int32_t mf_variant;                 /* MATRIX_FREE: the data path in use (ENS_MF_TILES / WARP /
                                           STAGED); 0 for the assembled kernels */
    int32_t comm_rank, comm_nranks;     /* NODE with nccl_comm: ncclCommUserRank / ncclCommCount of the
                                           communicator the halo runs on; -1 otherwise */
    int32_t mfs_consumers;              /* STAGED: consumer warps per CTA (0 otherwise) */
    int32_t mfs_unit_width;             /* STAGED: realisations per consumer unit (64 or 128) */
    int32_t mfs_stage_width;            /* STAGED: realisations per stage row (N_s, or the slice width
                                           of sliced stages) */
    int32_t mfs_stages;                 /* STAGED: shared-memory stages per CTA */
} ens_info;

/* Create a context: validate the mesh, build the RCM-ordered block-CSR pattern, the
 * element stiffnesses K^_e (E = 1, unit thickness, global frame), the Gauss-point
 * material scalings alpha_{e,s} = sum_g w_g E_g zeta_g, the lumped
 * masses, the central-difference coefficients and dt; upload; assemble the values on
 * the device (kernel = ASSEMBLED).  State starts at rest: u_0 = u_{-1} = 0, t = 0.
 * Traction starts at zero.  On error *out = NULL.  Collective when dist = NODE. */
int ens_create(const ens_mesh* mesh, const ens_materials* mat, const ens_options* opt, ens_ctx** out);

/* Prescribed wall traction, identical for all realisations (one-way coupling with a
 * rigid-wall fluid; loads applied as nodal forces):
 *   f(t) = ramp(t) * sum_k g_k(t) F_k,   ramp(t) = sin(pi t / (2 ramp_T)) for t < ramp_T, else 1
 *   (PAPER.md:512, 571), g_k = linear interpolation of tab_g[k][:] at tau = t mod period
 *   (period <= 0: no wrap), clamped to the end values; n_tab = 0 => g_k = 1.
 * F: [n_fields][V][3] nodal forces (dyn) in the caller's numbering, 1 <= n_fields <= 4.
 * tab_t: [n_tab] strictly increasing (s); tab_g: [n_fields][n_tab].  Copied before return.
 * The first call (or one changing n_fields or n_tab) allocates and synchronises; a later
 * call with the same shape packs the values into pinned staging and enqueues their copy on
 * the context stream after the steps already enqueued (asynchronous, no graph rebuild):
 * the per-window input update of a running simulation. */
int ens_set_traction(ens_ctx* ctx, int32_t n_fields, const double* F, int32_t n_tab,
                     const double* tab_t, const double* tab_g, double period, double ramp_T);

/* Enqueue n >= 0 fused steps on the context stream and return without waiting.  Each
 * step reads u_n, u_{n-1}, writes u_{n+1} over u_{n-1} and evaluates f at t_n = n dt.
 * A non-finite result sets a device flag that the next synchronising call
 * (ens_get_state / ens_sync) reports as ENS_E_DIVERGED; afterwards the context returns
 * ENS_E_STATE until ens_set_state. */
int ens_step(ens_ctx* ctx, int64_t n);

/* Build now what the first ens_step(n >= graph_steps) would otherwise build: the CUDA graphs
 * of the step loop for both parities of the starting step (capture + instantiate; no step is
 * executed and the state is untouched).  Setup work, so that a timed step loop does not pay
 * for it.  No-op without graphs (graph_steps == 0, persistent kernel,
 * re-assembly).  Collective with NCCL (the capture records the halo send/recv; a
 * communicator that cannot be captured makes every rank fall back to direct launches, as in
 * ens_step).  Errors: ENS_E_ARG (ctx NULL), ENS_E_STATE (P2P halo not connected),
 * ENS_E_CUDA. */
int ens_prepare(ens_ctx* ctx);

/* Wait for the enqueued work; report a pending divergence. */
int ens_sync(ens_ctx* ctx);

/* Snapshot of u_n without stopping the step loop (output every k steps):
 * enqueue, after the steps enqueued so far, the layout transpose of u_n on the context
 * stream and its device->host copy on a separate copy stream, then return.  u_n: caller
 * HOST buffer [n_s][R][3] as ens_get_state (pinned memory recommended: pageable memory makes
 * the copy synchronous); it must stay valid and untouched until ens_observe_wait returns.
 * One snapshot in flight: a second ens_observe orders its transpose after the previous
 * copy.  ens_observe_wait blocks until the copy is done, returns the snapshot's step, and
 * reports ENS_E_DIVERGED if a non-finite value had appeared by then (ENS_E_STATE if no
 * snapshot is in flight). */
int ens_observe(ens_ctx* ctx, double* u_n);
int ens_observe_wait(ens_ctx* ctx, int64_t* step);

/* Copy the state to caller-owned HOST buffers (either may be NULL):
 * u_n, u_nm1: [n_s][R][3] with R = V in the caller's node numbering, except for a NODE
 * context on NCCL, where R = the owned rows in the order ens_get_owned reports.
 * t, step may be NULL.  Synchronises the context. */
int ens_get_state(ens_ctx* ctx, double* u_n, double* u_nm1, double* t, int64_t* step);

/* Rows of ens_get_state / ens_apply_stiffness outputs: *n = R; node_ids[R] (may be NULL)
 * receives the caller node id of each row. */
int ens_get_owned(const ens_ctx* ctx, int32_t* node_ids, int64_t* n);

/* Overwrite the state (checkpoint / resume; clears the divergence latch).
 * u_n, u_nm1: FULL [n_s][V][3] host arrays in the caller's numbering (every rank of a NODE
 * group passes the full state: each takes its owned and ghost rows); NULL => zeros. */
int ens_set_state(ens_ctx* ctx, const double* u_n, const double* u_nm1, double t, int64_t step);

/* Diagnostic: y_s = K_s u_s for all s with the hot kernel's own product (same inner loop
 * and summation order as ens_step).  u: full [n_s][V][3]; y: [n_s][R][3] as ens_get_state. */
int ens_apply_stiffness(ens_ctx* ctx, const double* u, double* y);

/* Element stresses of u_n and their ensemble statistics (the step after the hot path,
 * SURVEY.md §8(f) N1).  Per element e and realisation s: eps = B T u_e (Eq. 8), sigma =
 * C(Ebar_{e,s}) eps (Eq. 7, 9; Ebar = element mean of the nodal E = the mean over the three
 * Gauss points).  frame 0: local shell frame, (s_xx, s_yy, t_xy, t_xz, t_yz, 0);
 * frame 1: the paper's frame: r = element normal, z = tangent of the
 * centreline polyline at its point closest to the centroid (orthogonalised to r),
 * theta = r x z; (s_rr, s_tt, s_zz, s_tz, s_rz, s_rt).  centerline [n_c][3] (n_c >= 2) or
 * NULL for the z axis.  Outputs (host, each may be NULL): sigma [n_s][F][6];
 * mean, q05, q95 [F][6] over the realisations: quantile p of the n
 * sorted values v is v[lo] + (h - lo)(v[lo+1] - v[lo]), h = (n-1) p, lo = floor(h).
 * Single-part contexts (not NODE on NCCL).  Synchronises. */
int ens_stress(ens_ctx* ctx, int32_t frame, const double* centerline, int32_t n_c, double* sigma,
               double* mean, double* q05, double* q95);

/* Ensemble statistics of u_n per node (caller numbering): mean, q05, q95 [V][4] =
 * (u_x, u_y, u_z, |u|), same quantile definition.  Single-part contexts.  Synchronises. */
int ens_displacement_stats(ens_ctx* ctx, double* mean, double* q05, double* q95);

/* GPU Matérn sampler (the step before the hot path): for each of the n
 * standard-normal vectors z[k][V] (caller numbering) returns the unit-variance GMRF draw
 *   x[k] = A^-1 C~^{1/2} z[k] / sigma,   A = kappa^2 C~ + G,   kappa = sqrt(8) / rho_corr,
 *   sigma^2 = 1 / (4 pi kappa^2)
 * (Matérn nu = 1, alpha = 2; Eqs. 2-6: covariance A^-1 C~ A^-1 = Q_2^-1,
 * the law of Eq. 11's Cholesky route).  C~: lumped P1 mass; G: P1
 * stiffness.  All n systems are solved together by Jacobi-preconditioned CG until every
 * relative residual <= tol (or max_iter).  *iters, *max_rel_res may be NULL.  opt supplies
 * device, stream and allocator (may be NULL).  Synchronous. */
int ens_matern_fields(const ens_mesh* mesh, double rho_corr, int32_t n, const double* z, double* x, double tol,
                      int32_t max_iter, const ens_options* opt, int32_t* iters, double* max_rel_res);

/* ---- ENS_HALO_P2P with one part per process (opt.p2p_procs = 1) ---------------------
 * ens_create allocates this part's state buffers and its neighbour flags with cudaMalloc
 * (IPC-exportable) and zeroes them.  ens_p2p_export writes ENS_P2P_BLOB_BYTES describing
 * them (CUDA IPC handles of u buffer 0, u buffer 1 and the flags, plus rank / world / row
 * counts) into blob.  The caller all-gathers the blobs of every rank over any host
 * channel (the Python binding uses torch.distributed) and passes the concatenation
 * blobs[world][ENS_P2P_BLOB_BYTES] to ens_p2p_connect, which opens the neighbours' buffers
 * (cudaIpcOpenMemHandle; peer access over NVLink when the devices differ) and checks their
 * sizes.  Collective: no rank may step before every rank has connected (the all-gather
 * orders this), and ens_set_state must be followed by a barrier before the next ens_step.
 * Errors: ENS_E_STATE (not such a context / already connected), ENS_E_ARG (blob of a
 * different world, rank or size), ENS_E_CUDA (IPC failure).  A neighbour that stops
 * stepping makes the waiting rank's flag wait time out after ~10 s; the next synchronising
 * call then returns ENS_E_CUDA naming the step and the neighbour. */
#define ENS_P2P_BLOB_BYTES 256
int ens_p2p_export(const ens_ctx* ctx, void* blob);
int ens_p2p_connect(ens_ctx* ctx, const void* blobs);

/* Measured FP64 FMA throughput of `device` (< 0: current), TFLOP/s: the ALU roofline the
 * matrix-free step is compared with (not in MEASURED_PEAKS.json).  A
 * DFMA loop with 8 independent chains per thread on 8 CTAs x 256 threads per SM, best of
 * 5 timed launches.  Synchronous; ENS_E_CUDA without a device. */
int ens_measure_fp64(int32_t device, double* tflops);

/* Sizes, dt and algorithmic traffic of the context. */
int ens_query(const ens_ctx* ctx, ens_info* info);

/* Destroy (NULL is a no-op).  Synchronises the stream first. */
void ens_destroy(ens_ctx* ctx);

/* Message of the last error on ctx (or, for ctx = NULL, of the last failed call on this
 * thread).  Valid until the next call on the same context / thread. */
const char* ens_last_error(const ens_ctx* ctx);

/* ---- host-side setup maps (no device needed; used by the CPU tests) ------------------ */

/* Mesh validation as in ens_create.  Returns ENS_OK or ENS_E_MESH; *bad = element (or the
 * first node of the offending edge).  *code: 1 index, 2 repeated node, 3 degenerate, 4 edge. */
int ens_host_validate(int64_t n_nodes, int64_t n_tris, const double* xyz, const int32_t* tris,
                      int32_t* code, int64_t* bad);

/* RCM permutation and block-CSR pattern exactly as ens_create builds them.
 * perm[V] (perm[new] = old), row_ptr[V+1], col[col_cap]; *nnzb = blocks written.
 * Returns ENS_E_ARG if col_cap is too small (*nnzb then holds the needed size). */
int ens_host_pattern(int64_t n_nodes, int64_t n_tris, const int32_t* tris, int32_t* perm,
                     int64_t* row_ptr, int32_t* col, int64_t col_cap, int64_t* nnzb);

/* Node-partition bounds (bounds[P+1]) of an RCM-ordered pattern, balanced by blocks. */
int ens_host_partition(int64_t n_nodes, const int64_t* row_ptr, int32_t n_parts, int64_t* bounds);

/* Ghost rows of part [lo, hi): sorted columns outside the range.  ghosts[cap]; *n = count. */
int ens_host_ghosts(int64_t n_nodes, const int64_t* row_ptr, const int32_t* col, int64_t lo,
                    int64_t hi, int32_t* ghosts, int64_t cap, int64_t* n);

/* Halo plan of part `part` of n_parts (as ens_create builds it for ENS_DIST_NODE):
 * lo_hi_b[5] = {lo, hi, b_lo, b_hi, n_ghost}: owned RCM rows [lo, hi); every row with a
 * ghost column is among local rows [0, b_lo) or [hi-lo-b_hi, hi-lo).  peers[n_parts] and
 * peer_info[n_parts][4] = {send_off, send_n, recv_row, recv_n} per neighbour (ascending
 * rank); send_rows[cap] = local rows sent, concatenated per neighbour. */
int ens_host_halo_plan(int64_t n_nodes, const int64_t* row_ptr, const int32_t* col, int32_t n_parts, int32_t part,
                       int64_t* lo_hi_b, int32_t* peers, int64_t* peer_info, int32_t* send_rows, int64_t cap,
                       int64_t* n_peers, int64_t* n_send);

/* Element stiffness K^_e (E = 1, unit thickness, global frame) and area, as ens_create
 * computes them.  Khat: [F][9][9]; area: [F]. */
int ens_host_element_stiffness(int64_t n_nodes, int64_t n_tris, const double* xyz,
                               const int32_t* tris, double nu, double k_shear, double* Khat,
                               double* area);

/* Gauss-point scaling alpha [n_s][F], lumped mass m [n_s][V] and CFL dt, as ens_create
 * computes them. */
int ens_host_materials(int64_t n_nodes, int64_t n_tris, const double* xyz, const int32_t* tris,
                       int32_t n_s, const double* E, const double* h, double rho,
                       double cfl_safety, double* alpha, double* mass, double* dt_cfl);

/* The matrix-free STAGED tiling of the whole RCM row range, as ens_create builds it for a
 * single-part context (kernels.cu k_step_mf_staged; DESIGN.md §5 F3): patches = 1 compact
 * patches / 0 strips of consecutive rows, at most max_rows rows per tile, stage_bytes = the
 * budget of one shared-memory stage (<= 0: the library's for this n_s).  Outputs: tile_of[V]
 * = the tile of each RCM row; tile_bytes[V] (first *n_tiles used) = blob + u_n + alpha bytes
 * of each tile (F_k excluded), tile_entries[V] = its bulk copies; *budget = the stage budget
 * used.  Host only. */
int ens_host_mf_tiles(int64_t n_nodes, int64_t n_tris, const double* xyz, const int32_t* tris, int32_t n_s,
                      int32_t patches, int32_t max_rows, int64_t stage_bytes, int32_t* tile_of,
                      int64_t* tile_bytes, int32_t* tile_entries, int64_t* n_tiles, int64_t* budget);

/* ---- test-only: synthetic operators (kernel unit tests, not the user contract) ----- */

/* A context on a caller-given block-CSR pattern (any numbering, used as is) and values:
 * row_ptr[V+1], col[nnzb], Kval[n_s][nnzb][9], c1/c2/c3 [n_s][V] (u_{n+1} =
 * c1 (f - K u) + c2 u_n - c3 u_{n-1}), fixed[V] or NULL. */
int ens_create_csr(int64_t n_nodes, const int64_t* row_ptr, const int32_t* col, int32_t n_s,
                   const double* Kval, const double* c1, const double* c2, const double* c3,
                   const uint8_t* fixed, double dt, const ens_options* opt, ens_ctx** out);

#ifdef __cplusplus
}
#endif
#endif /* ENS_H_ */
