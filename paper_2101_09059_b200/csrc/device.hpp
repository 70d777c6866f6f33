// device.hpp -- launchers of the sm_100a kernels (kernels.cu).  Device layout (DESIGN.md
// "HBM layout"): rows in RCM order, realisation innermost:
//   u      [V][3][n_s]      two ping-pong buffers; u_{n+1} overwrites u_{n-1}
//   Kval   [nnzb][9][n_s]   9 = (c, d) of the 3x3 node block, row-major
//   c1     [V][n_s]         (+ c2a, c3a [V][n_s] for damping = IDENTITY)
//   alpha  [F][n_s], Khat [F][81], etri [F][3] (RCM ids)
#pragma once

#include <cstdint>
#include <cuda_runtime_api.h>

namespace ens {

constexpr int kMaxFields = 4;
// kinds of the matrix-free item programs (StepArgs::items, kernels.cu F2w)
constexpr int kItemOwn = 0, kItemPrev = 1, kItemInc = 2, kItemOld = 3, kItemLastApply = 32;

// Matrix-free F3 (kernels.cu k_step_mf_staged): one tile = up to kMfsMaxRows rows (a compact
// patch of the mesh, grown greedily on the host) whose operands fit one shared-memory stage,
// laid out [blob | u_n | alpha | F_k]:
//   blob  = header int32[8] {nrows, u-image offset, row-offset offset, F_k offset, row-id
//           offset, 0, 0, 0} (byte offsets within the stage), then per incidence a 160-B
//           record (int4 {alpha byte offset, next-node byte offset, prev-node byte offset,
//           restart} + the 18 K^ coefficients of the (prev, next) columns), then int32 row
//           offsets [nrows + 1] into the records, each | (the row's Dirichlet bits << 24),
//           then int32 row ids [nrows]; padded to 128 B
//   u_n   = the tile's node set, its own rows first (tile order), each row [3][n_s] (n_s * 24 B)
//   alpha = the tile's elements, each row [n_s] (n_s * 8 B)
//   F_k   = the own rows' load fields, [n_fields][nrows][4] (32 B rows; n_fields is known
//           only at ens_set_traction, the host budgets kMaxFields)
// The stage is filled by the tile's COPY ENTRIES (one bulk copy each; int4 {kind, first,
// count, stage byte offset}): kMfsU u_n rows [first, first + count); kMfsA alpha rows;
// kMfsF own rows of every load field (offset + k * nrows * 32 for field k); kMfsBlob the
// blob (first = its offset in mfs_blob / 16, count = bytes).
constexpr int kMfsHdrBytes = 32;
constexpr int kMfsRecBytes = 160;
constexpr int kMfsMaxRows = 32;
#ifndef ENS_MFS_MAX_ENTRIES
#define ENS_MFS_MAX_ENTRIES 96
#endif
constexpr int kMfsMaxEntries = ENS_MFS_MAX_ENTRIES;   // copy entries per tile (32 per producer lane slot)
enum { kMfsU = 0, kMfsA = 1, kMfsF = 2, kMfsBlob = 3 };
struct MfTile {
    int32_t entry0, n_entries;    // copy entries [entry0, entry0 + n_entries) of mfs_entries
    int32_t nrows, stage_bytes;   // bytes of blob + u + alpha (+ F_k: n_fields * nrows * 32)
};

struct StepArgs {
    int64_t V = 0;            // rows handled by this launch: rows [row0, row0 + V)
    int64_t row0 = 0;
    int64_t fk_rows = 0;      // rows of the F_k arrays (the owned rows)
    int32_t n_s = 0;
    const int32_t* row_ptr = nullptr;   // [rows + 1] (int32: nnzb < 2^31)
    const int32_t* col = nullptr;
    const double* Kval = nullptr;
    // symmetric (half) block storage: Kval holds the stored blocks
    const int32_t* sym_lptr = nullptr;  // [rows + 1] lower references of each row
    const int32_t* sym_lidx = nullptr;  // stored block (j, i) used transposed by row i
    const int32_t* sym_lcol = nullptr;  // its column j (< i)
    const int2* sym_urange = nullptr;   // [rows] stored blocks (i, j >= i) of row i
    const int32_t* sym_scol = nullptr;  // [stored] column of each stored block
    // matrix-free operands (host_setup.hpp "Fans")
    const int32_t* inc_ptr = nullptr;   // [rows + 1] incidence range of each row
    const int4* fan = nullptr;          // [3F] {e, n_prev, n_next, restart}
    const double* Krow = nullptr;       // [3F][28]
    const double* alpha = nullptr;      // [F][n_s]
    int32_t mf_rows = 1;                // rows per CTA
    int32_t mf_groups = 1;              // realisation groups (threads) per row per CTA
    int32_t mf_smem_inc = 0;            // max incidences staged by one CTA
    int32_t mf_prefetch = 0;            // L2 prefetch distance in tiles (set by the launcher)
    // matrix-free item programs (kernels.cu F2w; built by capi.cpp when DIFF is on)
    const int32_t* item_ptr = nullptr;  // [rows + 1]
    const int4* items = nullptr;        // {node, elem | row, K^ row, kind | flags}
    // matrix-free tile stages (kernels.cu F3) of the launched row range
    const MfTile* mfs_tiles = nullptr;
    const int4* mfs_entries = nullptr;  // copy entries {kind, first, count, stage offset}
    const unsigned char* mfs_blob = nullptr;
    int32_t mfs_ntiles = 0;
    int32_t mfs_stage_bytes = 0;        // bytes per stage (shared memory = stages * this + barriers)
    int32_t mfs_shape = 0;              // consumer warps x stages (kernels.cu kMfsShapes)
    int32_t mfs_slices = 1;             // > 1: sliced stages (64 * WS realisations per stage row), N_s / (64 WS)
    int64_t mfs_alpha_rows = 0;         // rows of alpha (the part's elements; tensor maps)
    // update coefficients
    const double* c1 = nullptr;
    const double* c2a = nullptr;        // null => scalars c2, c3
    const double* c3a = nullptr;
    double c2 = 2.0, c3 = 1.0;
    const uint8_t* fixed = nullptr;     // [rows]
    // load f(t) = ramp(t) sum_k g_k(t) F_k
    int32_t n_fields = 0;
    const double* Fk = nullptr;         // [n_fields][fk_rows][4] (x, y, z, 0: 32 B rows for TMA)
    int32_t n_tab = 0;
    const double* tab_t = nullptr;      // device [n_tab]
    const double* tab_g = nullptr;      // device [n_fields][n_tab]
    double period = 0.0, ramp_T = 0.0, dt = 0.0;
    // time index: step = *step_base + step_off; u_n = buf[step & 1]
    const int64_t* step_base = nullptr;
    int64_t step_off = 0;
    double* ubuf0 = nullptr;
    double* ubuf1 = nullptr;
    int64_t u_rows = 0;                 // rows of each state buffer (owned + ghosts)
    unsigned long long* flag = nullptr; // min over (step << 24 | s) of non-finite results
    double* coef_buf = nullptr;         // [2][kMaxFields] load coefficients of steps of each parity
    int32_t s_global0 = 0;
    // diagnostic mode: y = K u_n written to y_out ([V][3][n_s]), no update
    double* y_out = nullptr;
    // P2P halo (ENS_HALO_P2P): u_{n+1} of local row i also goes to the neighbours' ghost rows
    // fwd_dst[fwd_ptr[i] .. fwd_ptr[i+1]) = {peer slot, row in the peer's local numbering};
    // peer_buf[2 slot + b] = the peer's state buffer b.  Null => no forwarding.
    const int32_t* fwd_ptr = nullptr;   // [rows + 1]
    const int2* fwd_dst = nullptr;
    double* const* peer_buf = nullptr;
    // P2P halo flags inside the step kernels (a1, a1s and F3): hw_wait =>
    // before any ghost row is read, every CTA waits until flags[in_q[k]] >= step for each of
    // the n_in neighbours (ld.acquire.sys, 10 s timeout -> *hw_err); hw_signal => the last CTA
    // of this launch to finish (counter *hw_done) publishes step + 1 to the n_out neighbours
    // (fence.sc.sys; st.release.sys).  Set on a part's first / last boundary-row launch, which
    // replace the separate k_halo_wait / k_halo_signal launches.
    int32_t hw_wait = 0, hw_signal = 0;
    const unsigned long long* hw_flags = nullptr;
    const int32_t* hw_in_q = nullptr;
    int32_t hw_n_in = 0, hw_n_out = 0;
    unsigned long long* const* hw_out = nullptr;
    unsigned int* hw_done = nullptr;
    unsigned long long* hw_err = nullptr;
};

// P2P halo: publish "ghost data of u_{step+1} stored" to every neighbour
// (out_flag[k] = the slot of this part in neighbour k's flag array; st.release.sys after a
// system fence), and wait until every neighbour q in in_q has published >= step
// (ld.acquire.sys on this part's own flags[q]).  step = *step_base + step_off.  A wait
// longer than ~10 s stores the step and neighbour into *herr and gives up.
cudaError_t launch_halo_signal(int32_t n_out, unsigned long long* const* out_flag, const int64_t* step_base,
                               int64_t step_off, cudaStream_t st);
cudaError_t launch_halo_wait(int32_t n_in, const int32_t* in_q, const unsigned long long* flags,
                             const int64_t* step_base, int64_t step_off, unsigned long long* herr, cudaStream_t st);

// Fused step (S2 load + S3 ensemble SpMM + S4 central-difference update) on the
// assembled values: one launch advances rows [row0, row0+V) by one step.
cudaError_t launch_step_assembled(const StepArgs& a, cudaStream_t st);
// Same on the symmetric half storage (blocks j >= i stored; bit-identical results).
cudaError_t launch_step_assembled_sym(const StepArgs& a, cudaStream_t st);
// Same on the matrix-free element form (alpha_{e,s} K^_e gathered per node).
cudaError_t launch_step_matrix_free(const StepArgs& a, cudaStream_t st);
// realisations per thread of the step kernels for a given N_s (4, 2 or 1)
int pick_vec(int32_t n_s);      // assembled kernel
int pick_vec_mf(int32_t n_s);   // matrix-free kernel
// matrix-free F3 (tile stages): applies to N_s % 64 == 0 with N_s / 64 <= consumer warps
bool mf_staged_applies(int32_t n_s);
// F3 launch shape: consumer warps, stages, and the stage byte budget of one tile
struct MfsShape { int consumers, stages, stage_bytes; };
MfsShape mf_staged_shape(int shape);
// per-context plan: shape index, tiling (patches or strips of consecutive rows), rows per tile
// sliced: a stage row holds one slice of 64 * ws realisations (ws = the shape's slices per unit)
struct MfsPlan { int shape = 0; bool patches = false; int max_rows = 16; bool sliced = false; int ws = 1; };
// realisations per stage row: the slice width when sliced, else N_s
inline int mfs_stage_w(const MfsPlan& p, int32_t n_s) { return p.sliced ? 64 * p.ws : int(n_s); }
MfsPlan mf_staged_plan(int32_t n_s);
bool mf_diff();            // matrix-free: neighbours relative to u_i, (prev, next) K^ columns only (ENS_MF_DIFF, default 1)
int mf_inc_bytes();        // matrix-free: shared-memory bytes per incidence (K^ image + fan record)
// coef_buf[(step & 1)] = the load coefficients of step *step_base (after host changes)
cudaError_t launch_seed_coeffs(const StepArgs& a, cudaStream_t st);
// FP64 FMA throughput of this device (TFLOP/s, best of 5 timed launches)
cudaError_t measure_fp64_fma(double* tflops);
// N2: n steps of every part in `parts` (device array of P StepArgs, items[P + 1] prefix of
// their (row, realisation group) counts) as one cooperative persistent launch of the a1
// (sym = false) or a1s kernel rows; flags != 0: one part per process, neighbour step flags
// waited for / published inside (parts[0].hw_*).  bar: [2] zeroed grid-barrier state.
cudaError_t launch_steps_persistent(const StepArgs* parts, const int64_t* items, int32_t P, int32_t n_s, bool sym,
                                    int64_t n, unsigned int* bar, int32_t flags, cudaStream_t st);
// *step_base += n (after n steps were enqueued)
cudaError_t launch_advance(int64_t* step_base, int64_t n, cudaStream_t st);

// F0: Kval[b][k][s] = sum_{(e, a, b') in contrib[b]} alpha[e][s] Khat[e][3a+c][3b'+d]
cudaError_t launch_assemble(int64_t nnzb, int32_t n_s, const int32_t* contrib_ptr, const int32_t* contrib,
                            const double* alpha, const double* Khat, double* Kval, cudaStream_t st);

// F4: device rows [rows][3][n_s] <-> ABI [n_s][V_abi][3] at node map[i]
cudaError_t launch_abi_to_dev(int64_t rows, int32_t n_s, const int32_t* map, int64_t V_abi, const double* src,
                              double* dst, cudaStream_t st);
cudaError_t launch_dev_to_abi(int64_t rows, int32_t n_s, const int32_t* map, int64_t V_abi, const double* src,
                              double* dst, cudaStream_t st);
// halo send-pack of u_{n+1} rows (step = *step_base + step_off)
cudaError_t launch_pack(int64_t n, int32_t n_s, const int32_t* rows, const int64_t* step_base, int64_t step_off,
                        const double* ubuf0, const double* ubuf1, double* sendbuf, cudaStream_t st);

}  // namespace ens
