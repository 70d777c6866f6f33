// host_setup.hpp -- one-time host setup of the ensemble shell solver (C++17).
//
// Everything the north star lists under "Host setup (done once)": mesh validation,
// mesh -> block-CSR pattern with RCM reordering, element stiffness K^_e, Gauss-point
// material scaling alpha_{e,s}, lumped mass, CFL step, node partition / halo maps.
// Independent of oracle/ (no shared code); integer maps are specified exactly in
// DESIGN.md "Pattern" so both reach the same bits.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace ens {

struct MeshView {
    int64_t V = 0, F = 0;
    const double* xyz = nullptr;    // [V][3]
    const int32_t* tris = nullptr;  // [F][3]
};

// 0 ok; 1 index out of range; 2 repeated node; 3 degenerate; 4 edge shared by > 2 triangles.
int validate_mesh(const MeshView& m, int64_t* bad);

struct Pattern {
    std::vector<int32_t> perm;      // perm[new] = old
    std::vector<int32_t> iperm;     // iperm[old] = new
    std::vector<int64_t> row_ptr;   // [V+1], RCM order
    std::vector<int32_t> col;       // [nnzb], ascending per row, diagonal included
    int32_t bandwidth = 0;
};

// Neighbour lists (sorted, unique, no self) of the triangulation's edge graph.
void edge_graph(const MeshView& m, std::vector<int64_t>& ptr, std::vector<int32_t>& adj);
std::vector<int32_t> rcm_order(int64_t V, const std::vector<int64_t>& ptr, const std::vector<int32_t>& adj);
Pattern build_pattern(const MeshView& m);

// K^_e for E = 1 and unit thickness in the global frame (81 doubles) + area.
void element_stiffness(const double* X1, const double* X2, const double* X3, double nu,
                       double k_shear, double* Khat, double* area);

// Strain operator of element (X1, X2, X3): eps_local[5] = G[5][9] u_global[9] (Eq. 8 with
// the frame rotation folded in), and R[3][3] = the local basis (rows e1, e2, e3).
void element_strain_operator(const double* X1, const double* X2, const double* X3, double* G, double* R);

// Output basis of the stress recovery expressed in the local basis:
// frame 0: identity; frame 1: rows (r, theta, z) with r = e3, z = the centreline tangent
// closest to the centroid made orthogonal to r, theta = r x z.  M[3][3] = b R^T.
void stress_frame(const double* centroid, const double* R, int32_t frame, const double* centerline,
                  int32_t n_c, double* M);

// alpha[s][e] (closed form of the 3-point Gauss rule on P1 fields), mass[s][v], CFL dt.
void materials(const MeshView& m, int32_t n_s, const double* E, const double* h, double rho,
               double* alpha, double* mass);
double cfl_dt(const MeshView& m, int32_t n_s, const double* E, double rho, double safety);

// SPDE/GMRF system on the wall mesh (N3): scalar CSR values of A = kappa^2 C~ + G on the
// pattern (RCM order), with C~ the lumped P1 mass and G_ab = e_a . e_b / (4 A_e)
// (e_a the edge opposite vertex a; Eq. 5-6); diag(A) and C~ per row.
void gmrf_system(const MeshView& m, const Pattern& pat, double kappa, std::vector<double>& val,
                 std::vector<double>& diag, std::vector<double>& lumped);

// Matrix-free operator arranged for the node-centric gather: for each
// row i (RCM order) its incident elements as chains of a fan around i, so that consecutive
// incidences (i, p_k, p_k+1), (i, p_k+1, p_k+2) share the node p_k+1.
struct FanRec {
    int32_t e;        // element (alpha row)
    int32_t n_prev;   // p_k   (RCM id)
    int32_t n_next;   // p_k+1 (RCM id)
    int32_t restart;  // 1: first incidence of a chain (n_prev must be loaded)
};
struct Fans {
    std::vector<int32_t> ptr;     // [V+1] incidence range of each row
    std::vector<FanRec> rec;      // [3F]
    std::vector<double> Krow;     // [3F][28]: K^_e rows 3a..3a+2, columns (own, p_k, p_k+1) x 3, + pad
};
Fans build_fans(const MeshView& m, const std::vector<int32_t>& iperm, const std::vector<double>& Khat);

// Node partition of the RCM rows balanced by blocks, and ghost rows.
std::vector<int64_t> partition_bounds(const std::vector<int64_t>& row_ptr, int32_t P);
std::vector<int32_t> ghost_rows(const std::vector<int64_t>& row_ptr, const std::vector<int32_t>& col,
                                int64_t lo, int64_t hi);

// Halo plan of part p.  Local rows: the owned rows
// [lo, hi) in global order, then the ghosts in ascending global order (hence grouped by
// owner: each neighbour's ghosts are one contiguous slice, received in place).
struct PartPlan {
    int32_t p = 0;
    int64_t lo = 0, hi = 0;
    std::vector<int32_t> ghosts;        // global RCM ids, ascending
    int64_t b_lo = 0, b_hi = 0;         // every row with a ghost column lies in local rows
                                        // [0, b_lo) or [n_own - b_hi, n_own)
    struct Peer {
        int32_t q = 0;
        int64_t send_off = 0, send_n = 0;   // slice of send_rows / the send buffer
        int64_t recv_row = 0, recv_n = 0;   // local row of the first ghost owned by q
    };
    std::vector<Peer> peers;            // ascending q
    std::vector<int32_t> send_rows;     // local owned rows, concatenated per peer
    int64_t n_own() const { return hi - lo; }
};
std::vector<PartPlan> halo_plan(const std::vector<int64_t>& row_ptr, const std::vector<int32_t>& col, int32_t P);

}  // namespace ens
