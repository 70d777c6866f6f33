/*
 * oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the ensemble explicit
 * shell solver of arXiv 2101.09059 ("PAPER.md" below = /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code with
 * the CUDA path (paper_2101_09059_b200/csrc, include/ens.h) and includes none of its
 * headers.  Compiled with -O2 -ffp-contract=off (no FMA contraction) so every
 * expression is evaluated exactly as written.
 *
 * Conventions
 *   - Node numbering is the caller's ORIGINAL numbering (no reordering) for all of the
 *     dynamics; the RCM ordering (orc_rcm) exists only so tests can compare the CUDA
 *     path's integer maps against it.
 *   - Ensemble arrays are realisation-OUTERMOST: u[s][node][3], Kval[s][block][3][3],
 *     alpha[s][elem], m[s][node]: each realisation is literally an independent solve
 *     ("no approximation introduced").
 *   - Readings of silent/ambiguous passages: SURVEY.md §8(c) C13, listed in DESIGN.md.
 *
 * Parity status: every function below is pinned by tests/test_oracle_*.py (DESIGN.md
 * "Oracle pins"); none is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------ */
/* Mesh validation (ABI contract include/ens.h).                     */
/* Returns 0 ok, 1 node index out of range, 2 repeated node in a triangle,               */
/* 3 zero-area triangle, 4 an edge shared by more than two triangles.                   */
/* *bad receives the offending element (codes 1-3) or the first node of the edge (4).   */
/* ------------------------------------------------------------------------------------ */

static int cmp_pair(const void* a, const void* b) {
    const int64_t* x = (const int64_t*)a;
    const int64_t* y = (const int64_t*)b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;
    return 0;
}

static double tri_area(const double* X1, const double* X2, const double* X3) {
    double a[3] = {X2[0] - X1[0], X2[1] - X1[1], X2[2] - X1[2]};
    double b[3] = {X3[0] - X1[0], X3[1] - X1[1], X3[2] - X1[2]};
    double n[3] = {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
    return 0.5 * sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
}

int orc_validate_mesh(int64_t V, int64_t F, const double* xyz, const int32_t* tris, int64_t* bad) {
    *bad = -1;
    for (int64_t e = 0; e < F; e++) {
        for (int a = 0; a < 3; a++)
            if (tris[3 * e + a] < 0 || tris[3 * e + a] >= V) { *bad = e; return 1; }
        int32_t p = tris[3 * e], q = tris[3 * e + 1], r = tris[3 * e + 2];
        if (p == q || q == r || p == r) { *bad = e; return 2; }
        /* degenerate: A_e <= 1e-12 * (sum of squared edge lengths) (scale-free "A_e > 0") */
        const double *P = xyz + 3 * (int64_t)p, *Q = xyz + 3 * (int64_t)q, *R = xyz + 3 * (int64_t)r;
        double l2 = 0.0;
        for (int c = 0; c < 3; c++)
            l2 += (Q[c] - P[c]) * (Q[c] - P[c]) + (R[c] - Q[c]) * (R[c] - Q[c]) + (P[c] - R[c]) * (P[c] - R[c]);
        if (!(tri_area(P, Q, R) > 1e-12 * l2)) { *bad = e; return 3; }
    }
    int64_t* pairs = (int64_t*)malloc(sizeof(int64_t) * 2 * 3 * (F > 0 ? F : 1));
    for (int64_t e = 0; e < F; e++)
        for (int a = 0; a < 3; a++) {
            int64_t p = tris[3 * e + a], q = tris[3 * e + (a + 1) % 3];
            pairs[2 * (3 * e + a)] = p < q ? p : q;
            pairs[2 * (3 * e + a) + 1] = p < q ? q : p;
        }
    qsort(pairs, (size_t)(3 * F), 2 * sizeof(int64_t), cmp_pair);
    int rc = 0;
    for (int64_t k = 0; k + 2 < 3 * F; k++)
        if (cmp_pair(pairs + 2 * k, pairs + 2 * (k + 2)) == 0) { *bad = pairs[2 * k]; rc = 4; break; }
    free(pairs);
    if (rc) return rc;
    /* a node in no triangle has lumped mass 0 (m_i = rho sum_e A_e zeta/3), */
    /* the divisor of Eq. 22's update: rejected                                           */
    char* used = (char*)calloc((size_t)(V > 0 ? V : 1), 1);
    for (int64_t k = 0; k < 3 * F; k++) used[tris[k]] = 1;
    for (int64_t i = 0; i < V; i++)
        if (!used[i]) { *bad = i; rc = 5; break; }
    free(used);
    return rc;
}

/* ------------------------------------------------------------------------------------ */
/* Node adjacency (one-ring) of the triangulation.  The stiffness couples node i to     */
/* node j iff they share a triangle ("immediate neighbors"; the 3x3-block   */
/* CSR of PAPER.md:349).  adj_ptr[V+1], adj[cap >= 6F]; neighbours ascending, no self.  */
/* Returns the number of directed neighbour entries (= 2 * #edges).                     */
/* ------------------------------------------------------------------------------------ */
int64_t orc_adjacency(int64_t V, int64_t F, const int32_t* tris, int64_t* adj_ptr, int32_t* adj) {
    int64_t n = 6 * F;
    int64_t* pairs = (int64_t*)malloc(sizeof(int64_t) * 2 * (n > 0 ? n : 1));
    int64_t k = 0;
    for (int64_t e = 0; e < F; e++)
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++)
                if (a != b) {
                    pairs[2 * k] = tris[3 * e + a];
                    pairs[2 * k + 1] = tris[3 * e + b];
                    k++;
                }
    qsort(pairs, (size_t)n, 2 * sizeof(int64_t), cmp_pair);
    for (int64_t i = 0; i <= V; i++) adj_ptr[i] = 0;
    int64_t m = 0;
    for (int64_t t = 0; t < n; t++) {
        if (t > 0 && cmp_pair(pairs + 2 * t, pairs + 2 * (t - 1)) == 0) continue;
        adj[m++] = (int32_t)pairs[2 * t + 1];
        adj_ptr[pairs[2 * t] + 1]++;
    }
    for (int64_t i = 0; i < V; i++) adj_ptr[i + 1] += adj_ptr[i];
    free(pairs);
    return m;
}

/* ------------------------------------------------------------------------------------ */
/* Reverse Cuthill-McKee ordering, fully specified so that two     */
/* independent implementations agree bit for bit.  The paper partitions with parMETIS  */
/* (PAPER.md:427); this deterministic ordering replaces it.                 */
/*   1. components in order of their lowest original index;                            */
/*   2. start node: George-Liu pseudo-peripheral search from the component's minimum-  */
/*      degree node (ties -> lowest index): BFS, take the minimum-degree node of the    */
/*      last level (ties -> lowest index); if its eccentricity is larger, move there   */
/*      and repeat, else keep the current node;                                         */
/*   3. Cuthill-McKee BFS: each dequeued node enqueues its unvisited neighbours sorted  */
/*      by (degree ascending, original index ascending);                                */
/*   4. reverse the whole concatenated order.  perm[new] = old.                         */
/* ------------------------------------------------------------------------------------ */

/* BFS from r over the whole graph; returns eccentricity, fills the last level. */
static int64_t bfs_levels(int64_t V, const int64_t* adj_ptr, const int32_t* adj, int64_t r,
                          int64_t* level, int64_t* queue, int64_t* last, int64_t* n_last) {
    for (int64_t i = 0; i < V; i++) level[i] = -1;
    int64_t head = 0, tail = 0;
    queue[tail++] = r;
    level[r] = 0;
    int64_t ecc = 0;
    while (head < tail) {
        int64_t v = queue[head++];
        for (int64_t k = adj_ptr[v]; k < adj_ptr[v + 1]; k++) {
            int64_t w = adj[k];
            if (level[w] < 0) {
                level[w] = level[v] + 1;
                if (level[w] > ecc) ecc = level[w];
                queue[tail++] = w;
            }
        }
    }
    *n_last = 0;
    for (int64_t t = 0; t < tail; t++)
        if (level[queue[t]] == ecc) last[(*n_last)++] = queue[t];
    return ecc;
}

static const int64_t* g_deg; /* for the qsort comparator below */
static int cmp_deg_idx(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    if (g_deg[x] != g_deg[y]) return g_deg[x] < g_deg[y] ? -1 : 1;
    return x < y ? -1 : (x > y ? 1 : 0);
}

void orc_rcm(int64_t V, const int64_t* adj_ptr, const int32_t* adj, int32_t* perm) {
    int64_t* deg = (int64_t*)malloc(sizeof(int64_t) * (V + 1));
    int64_t* level = (int64_t*)malloc(sizeof(int64_t) * (V + 1));
    int64_t* queue = (int64_t*)malloc(sizeof(int64_t) * (V + 1));
    int64_t* last = (int64_t*)malloc(sizeof(int64_t) * (V + 1));
    int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (V + 1));
    int64_t* nb = (int64_t*)malloc(sizeof(int64_t) * (V + 1));
    char* visited = (char*)calloc((size_t)V + 1, 1);
    for (int64_t i = 0; i < V; i++) deg[i] = adj_ptr[i + 1] - adj_ptr[i];
    g_deg = deg;
    int64_t pos = 0;
    for (int64_t c0 = 0; c0 < V; c0++) {
        if (visited[c0]) continue;
        /* component of c0 = the BFS tree from c0 */
        int64_t n_last, ecc;
        bfs_levels(V, adj_ptr, adj, c0, level, queue, last, &n_last);
        int64_t r = -1;
        for (int64_t i = 0; i < V; i++)
            if (level[i] >= 0 && (r < 0 || deg[i] < deg[r])) r = i; /* ascending i => lowest index on ties */
        ecc = bfs_levels(V, adj_ptr, adj, r, level, queue, last, &n_last);
        for (;;) {
            int64_t x = -1;
            for (int64_t t = 0; t < n_last; t++)
                if (x < 0 || deg[last[t]] < deg[x] || (deg[last[t]] == deg[x] && last[t] < x)) x = last[t];
            int64_t n_last_x;
            int64_t* last_x = (int64_t*)malloc(sizeof(int64_t) * (V + 1));
            int64_t ecc_x = bfs_levels(V, adj_ptr, adj, x, level, queue, last_x, &n_last_x);
            if (ecc_x > ecc) {
                r = x;
                ecc = ecc_x;
                memcpy(last, last_x, sizeof(int64_t) * n_last_x);
                n_last = n_last_x;
                free(last_x);
            } else {
                free(last_x);
                break;
            }
        }
        /* Cuthill-McKee from r */
        int64_t head = pos;
        order[pos++] = r;
        visited[r] = 1;
        while (head < pos) {
            int64_t v = order[head++];
            int64_t cnt = 0;
            for (int64_t k = adj_ptr[v]; k < adj_ptr[v + 1]; k++)
                if (!visited[adj[k]]) nb[cnt++] = adj[k];
            qsort(nb, (size_t)cnt, sizeof(int64_t), cmp_deg_idx);
            for (int64_t t = 0; t < cnt; t++) {
                visited[nb[t]] = 1;
                order[pos++] = nb[t];
            }
        }
    }
    for (int64_t i = 0; i < V; i++) perm[i] = (int32_t)order[V - 1 - i];
    free(deg); free(level); free(queue); free(last); free(order); free(nb); free(visited);
}

/* ------------------------------------------------------------------------------------ */
/* Block CSR pattern ("Yale" CSR with 3x3 node blocks).  Row i (new       */
/* numbering) holds node perm[i]; its columns are {i} U {new ids of its neighbours},     */
/* ascending.  iperm[old] = new.  Pass perm = NULL for the original numbering.          */
/* Returns nnzb.                                                                        */
/* ------------------------------------------------------------------------------------ */
static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

int64_t orc_csr(int64_t V, const int64_t* adj_ptr, const int32_t* adj, const int32_t* perm,
                int64_t* row_ptr, int32_t* col) {
    int32_t* iperm = (int32_t*)malloc(sizeof(int32_t) * (V + 1));
    for (int64_t i = 0; i < V; i++) iperm[perm ? perm[i] : i] = (int32_t)i;
    row_ptr[0] = 0;
    for (int64_t i = 0; i < V; i++) {
        int64_t old = perm ? perm[i] : i;
        int64_t p = row_ptr[i];
        col[p++] = (int32_t)i;
        for (int64_t k = adj_ptr[old]; k < adj_ptr[old + 1]; k++) col[p++] = iperm[adj[k]];
        qsort(col + row_ptr[i], (size_t)(p - row_ptr[i]), sizeof(int32_t), cmp_i32);
        row_ptr[i + 1] = p;
    }
    free(iperm);
    return row_ptr[V];
}

/* ------------------------------------------------------------------------------------ */
/* Element stiffness of the 3-dof linear membrane + transverse-shear shell, for E = 1,  */
/* unit thickness, in the GLOBAL frame:                             */
/*   local frame: e1 = (X2-X1)/|X2-X1|, e3 = unit normal, e2 = e3 x e1;   */
/*   local coords x_a = (X_a-X1).e1, y_a = (X_a-X1).e2;                                 */
/*   B  = Eq. 8, 5x9 with the 1/(2 A_e) factor;                       */
/*   C^ = Eq. 9 with E = 1;                                          */
/*   k^l = A_e B^T C^ B  (Eq. 10, for E zeta = 1);                         */
/*   K^  = T^T k^l T, T = diag(R,R,R), R = [e1; e2; e3] (rows).                          */
/* The upper triangle is mirrored so K^ is exactly symmetric.                           */
/* ------------------------------------------------------------------------------------ */
void orc_element_khat(const double* X, double nu, double kshear, double* Khat, double* area) {
    const double* X1 = X;
    const double* X2 = X + 3;
    const double* X3 = X + 6;
    double d21[3], d31[3], n[3], e1[3], e2[3], e3[3];
    for (int c = 0; c < 3; c++) { d21[c] = X2[c] - X1[c]; d31[c] = X3[c] - X1[c]; }
    n[0] = d21[1] * d31[2] - d21[2] * d31[1];
    n[1] = d21[2] * d31[0] - d21[0] * d31[2];
    n[2] = d21[0] * d31[1] - d21[1] * d31[0];
    double nn = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
    double A = 0.5 * nn;
    double l21 = sqrt(d21[0] * d21[0] + d21[1] * d21[1] + d21[2] * d21[2]);
    for (int c = 0; c < 3; c++) { e1[c] = d21[c] / l21; e3[c] = n[c] / nn; }
    e2[0] = e3[1] * e1[2] - e3[2] * e1[1];
    e2[1] = e3[2] * e1[0] - e3[0] * e1[2];
    e2[2] = e3[0] * e1[1] - e3[1] * e1[0];

    double x[3], y[3];
    for (int a = 0; a < 3; a++) {
        const double* Xa = X + 3 * a;
        double d[3] = {Xa[0] - X1[0], Xa[1] - X1[1], Xa[2] - X1[2]};
        x[a] = d[0] * e1[0] + d[1] * e1[1] + d[2] * e1[2];
        y[a] = d[0] * e2[0] + d[1] * e2[1] + d[2] * e2[2];
    }
    /* x_ij = x_i - x_j (1-based in the paper) */
    double y23 = y[1] - y[2], y31 = y[2] - y[0], y12 = y[0] - y[1];
    double x32 = x[2] - x[1], x13 = x[0] - x[2], x21 = x[1] - x[0];
    double Bm[5][9];
    memset(Bm, 0, sizeof(Bm));
    double f = 1.0 / (2.0 * A);
    /* row 0: eps_xx */
    Bm[0][0] = y23; Bm[0][3] = y31; Bm[0][6] = y12;
    /* row 1: eps_yy */
    Bm[1][1] = x32; Bm[1][4] = x13; Bm[1][7] = x21;
    /* row 2: gamma_xy */
    Bm[2][0] = x32; Bm[2][1] = y23; Bm[2][3] = x13; Bm[2][4] = y31; Bm[2][6] = x21; Bm[2][7] = y12;
    /* row 3: du_z/dx */
    Bm[3][2] = y23; Bm[3][5] = y31; Bm[3][8] = y12;
    /* row 4: du_z/dy */
    Bm[4][2] = x32; Bm[4][5] = x13; Bm[4][8] = x21;
    for (int r = 0; r < 5; r++)
        for (int c = 0; c < 9; c++) Bm[r][c] = Bm[r][c] * f;

    double Ch[5][5];
    memset(Ch, 0, sizeof(Ch));
    double pre = 1.0 / (1.0 - nu * nu);
    Ch[0][0] = pre;      Ch[0][1] = pre * nu;
    Ch[1][0] = pre * nu; Ch[1][1] = pre;
    Ch[2][2] = pre * 0.5 * (1.0 - nu);
    Ch[3][3] = pre * 0.5 * kshear * (1.0 - nu);
    Ch[4][4] = pre * 0.5 * kshear * (1.0 - nu);

    /* k^l = A * B^T C^ B */
    double CB[5][9], kl[9][9];
    for (int r = 0; r < 5; r++)
        for (int c = 0; c < 9; c++) {
            double s = 0.0;
            for (int m = 0; m < 5; m++) s += Ch[r][m] * Bm[m][c];
            CB[r][c] = s;
        }
    for (int i = 0; i < 9; i++)
        for (int j = 0; j < 9; j++) {
            double s = 0.0;
            for (int m = 0; m < 5; m++) s += Bm[m][i] * CB[m][j];
            kl[i][j] = A * s;
        }
    /* T (9x9) = diag(R,R,R); u_local = T u_global; K^ = T^T k^l T */
    double T[9][9];
    memset(T, 0, sizeof(T));
    for (int a = 0; a < 3; a++)
        for (int c = 0; c < 3; c++) {
            T[3 * a + 0][3 * a + c] = e1[c];
            T[3 * a + 1][3 * a + c] = e2[c];
            T[3 * a + 2][3 * a + c] = e3[c];
        }
    double kT[9][9];
    for (int i = 0; i < 9; i++)
        for (int j = 0; j < 9; j++) {
            double s = 0.0;
            for (int m = 0; m < 9; m++) s += kl[i][m] * T[m][j];
            kT[i][j] = s;
        }
    for (int i = 0; i < 9; i++)
        for (int j = i; j < 9; j++) {
            double s = 0.0;
            for (int m = 0; m < 9; m++) s += T[m][i] * kT[m][j];
            Khat[9 * i + j] = s;
            Khat[9 * j + i] = s;
        }
    *area = A;
}

void orc_all_khat(int64_t F, const double* xyz, const int32_t* tris, double nu, double kshear,
                  double* Khat, double* area) {
    for (int64_t e = 0; e < F; e++) {
        double X[9];
        for (int a = 0; a < 3; a++)
            for (int c = 0; c < 3; c++) X[3 * a + c] = xyz[3 * (int64_t)tris[3 * e + a] + c];
        orc_element_khat(X, nu, kshear, Khat + 81 * e, area + e);
    }
}

/* ------------------------------------------------------------------------------------ */
/* Material scaling per element and realisation:                   */
/*   k_e = sum_g B^T C(E_g) B A_e zeta_g w_g  (Eq. 10) = alpha_e K^_e      */
/*   alpha_{e,s} = sum_g w_g E_s(g) zeta_s(g),  w_g = 1/3,                               */
/* three-point rule at barycentric (2/3,1/6,1/6) and permutations, E and zeta P1-       */
/* interpolated from the nodal draws ("linear variation ... through each element",      */
/* PAPER.md:206).  E, h: [n_s][V]; alpha: [n_s][F].                                      */
/* ------------------------------------------------------------------------------------ */
void orc_alpha(int64_t V, int64_t F, const int32_t* tris, int32_t n_s, const double* E,
               const double* h, double* alpha) {
    static const double lam[3][3] = {{2.0 / 3.0, 1.0 / 6.0, 1.0 / 6.0},
                                     {1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0},
                                     {1.0 / 6.0, 1.0 / 6.0, 2.0 / 3.0}};
    for (int32_t s = 0; s < n_s; s++)
        for (int64_t e = 0; e < F; e++) {
            double sum = 0.0;
            for (int g = 0; g < 3; g++) {
                double Eg = 0.0, hg = 0.0;
                for (int a = 0; a < 3; a++) {
                    int64_t node = tris[3 * e + a];
                    Eg += lam[g][a] * E[(int64_t)s * V + node];
                    hg += lam[g][a] * h[(int64_t)s * V + node];
                }
                sum += (1.0 / 3.0) * Eg * hg;
            }
            alpha[(int64_t)s * F + e] = sum;
        }
}

/* ------------------------------------------------------------------------------------ */
/* Assembly of the per-realisation block values ("pre-assembled",   */
/* "dense coefficient entries of size 9 n_s"):                         */
/*   Kval_s[i,j][c][d] = sum_{e containing i and j, ascending e} alpha_{e,s} K^_e[3a+c][3b+d] */
/* with a, b the local indices of i, j in e.  Pattern in the caller's numbering          */
/* (row_ptr/col from orc_csr with perm = NULL).  Kval: [n_s][nnzb][9].                   */
/* ------------------------------------------------------------------------------------ */
static int64_t find_block(const int64_t* row_ptr, const int32_t* col, int64_t i, int64_t j) {
    for (int64_t b = row_ptr[i]; b < row_ptr[i + 1]; b++)
        if (col[b] == j) return b;
    return -1;
}

int orc_assemble(int64_t V, int64_t F, const int32_t* tris, const int64_t* row_ptr,
                 const int32_t* col, const double* Khat, int32_t n_s, const double* alpha,
                 double* Kval) {
    int64_t nnzb = row_ptr[V];
    for (int32_t s = 0; s < n_s; s++) {
        double* K = Kval + (int64_t)s * nnzb * 9;
        for (int64_t t = 0; t < nnzb * 9; t++) K[t] = 0.0;
        for (int64_t e = 0; e < F; e++) {
            double al = alpha[(int64_t)s * F + e];
            for (int a = 0; a < 3; a++)
                for (int b = 0; b < 3; b++) {
                    int64_t blk = find_block(row_ptr, col, tris[3 * e + a], tris[3 * e + b]);
                    if (blk < 0) return -1;
                    for (int c = 0; c < 3; c++)
                        for (int d = 0; d < 3; d++)
                            K[blk * 9 + 3 * c + d] += al * Khat[81 * e + 9 * (3 * a + c) + (3 * b + d)];
                }
        }
    }
    return 0;
}

/* ------------------------------------------------------------------------------------ */
/* Lumped mass per node and realisation ("lumped  */
/* mass matrix pre-assembled before the beginning of the time loop"):                    */
/*   m_{i,s} = rho * sum_{e containing i} A_e * zetabar_{e,s} / 3,                       */
/*   zetabar = mean of the three nodal thicknesses.  m: [n_s][V].                        */
/* ------------------------------------------------------------------------------------ */
void orc_mass(int64_t V, int64_t F, const double* xyz, const int32_t* tris, int32_t n_s,
              const double* h, double rho, double* m) {
    for (int32_t s = 0; s < n_s; s++) {
        for (int64_t i = 0; i < V; i++) m[(int64_t)s * V + i] = 0.0;
        for (int64_t e = 0; e < F; e++) {
            const int32_t* t = tris + 3 * e;
            double A = tri_area(xyz + 3 * (int64_t)t[0], xyz + 3 * (int64_t)t[1], xyz + 3 * (int64_t)t[2]);
            double hb = (h[(int64_t)s * V + t[0]] + h[(int64_t)s * V + t[1]] + h[(int64_t)s * V + t[2]]) / 3.0;
            double me = rho * A * hb / 3.0;
            for (int a = 0; a < 3; a++) m[(int64_t)s * V + t[a]] += me;
        }
    }
}

/* ------------------------------------------------------------------------------------ */
/* Central-difference coefficients (Eq. 22; lumped M~ and C~,          */
/* PAPER.md:341; f_v = -c_d u'; readings SURVEY.md C13 #3-#4):             */
/*   D = m + dt c / 2,  c1 = dt^2 / D,  c2 = 2 m / D,  c3 = (m - dt c / 2) / D          */
/* damping 0: c = 0;  1: c = c_d m (C~ = c_d M~);  2: c = c_d (C~ = c_d I).              */
/* so that u_{n+1} = c1 (f_n - K u_n) + c2 u_n - c3 u_{n-1}.  Arrays [n_s][V].           */
/* ------------------------------------------------------------------------------------ */
void orc_coeffs(int64_t V, int32_t n_s, const double* m, double dt, int32_t damping, double c_d,
                double* c1, double* c2, double* c3) {
    for (int64_t t = 0; t < (int64_t)n_s * V; t++) {
        double c = 0.0;
        if (damping == 1) c = c_d * m[t];
        if (damping == 2) c = c_d;
        double D = m[t] + dt * c / 2.0;
        c1[t] = dt * dt / D;
        c2[t] = 2.0 * m[t] / D;
        c3[t] = (m[t] - dt * c / 2.0) / D;
    }
}

/* ------------------------------------------------------------------------------------ */
/* CFL time step: d_e = 4 A_e / perimeter_e (diameter of  */
/* the inscribed circle), c = sqrt(E_max / rho) with E_max the largest Gauss-point E    */
/* over all elements and realisations; dt = safety * min_e d_e / c.                      */
/* ------------------------------------------------------------------------------------ */
double orc_cfl(int64_t V, int64_t F, const double* xyz, const int32_t* tris, int32_t n_s,
               const double* E, double rho, double safety) {
    double dmin = INFINITY, Emax = 0.0;
    for (int64_t e = 0; e < F; e++) {
        const double* P[3];
        for (int a = 0; a < 3; a++) P[a] = xyz + 3 * (int64_t)tris[3 * e + a];
        double per = 0.0;
        for (int a = 0; a < 3; a++) {
            const double* p = P[a];
            const double* q = P[(a + 1) % 3];
            per += sqrt((q[0] - p[0]) * (q[0] - p[0]) + (q[1] - p[1]) * (q[1] - p[1]) + (q[2] - p[2]) * (q[2] - p[2]));
        }
        double d = 4.0 * tri_area(P[0], P[1], P[2]) / per;
        if (d < dmin) dmin = d;
    }
    static const double lam[3][3] = {{2.0 / 3.0, 1.0 / 6.0, 1.0 / 6.0},
                                     {1.0 / 6.0, 2.0 / 3.0, 1.0 / 6.0},
                                     {1.0 / 6.0, 1.0 / 6.0, 2.0 / 3.0}};
    for (int32_t s = 0; s < n_s; s++)
        for (int64_t e = 0; e < F; e++)
            for (int g = 0; g < 3; g++) {
                double Eg = 0.0;
                for (int a = 0; a < 3; a++) Eg += lam[g][a] * E[(int64_t)s * V + tris[3 * e + a]];
                if (Eg > Emax) Emax = Eg;
            }
    return safety * dmin / sqrt(Emax / rho);
}

/* ------------------------------------------------------------------------------------ */
/* Load coefficients at time t (ens_set_traction contract):           */
/*   coef_k = ramp(t) * g_k(t),  ramp(t) = sin(pi t / (2 T_r)) for t < T_r else 1,       */
/*   g_k = piecewise-linear interpolation of tab_g[k][:] at tau = t mod period          */
/*   (no wrap if period <= 0), clamped at the table ends; n_tab = 0 => g_k = 1.          */
/* ------------------------------------------------------------------------------------ */
void orc_load_coeffs(double t, int32_t K, int32_t n_tab, const double* tab_t,
                     const double* tab_g, double period, double ramp_T, double* coef) {
    double ramp = 1.0;
    if (ramp_T > 0.0 && t < ramp_T) ramp = sin(M_PI * t / (2.0 * ramp_T));
    double tau = t;
    if (period > 0.0) tau = t - period * floor(t / period);
    for (int32_t k = 0; k < K; k++) {
        double g = 1.0;
        if (n_tab > 0) {
            const double* G = tab_g + (int64_t)k * n_tab;
            if (tau <= tab_t[0]) g = G[0];
            else if (tau >= tab_t[n_tab - 1]) g = G[n_tab - 1];
            else {
                int32_t j = 0;
                while (!(tab_t[j] <= tau && tau < tab_t[j + 1])) j++;
                g = G[j] + (G[j + 1] - G[j]) * (tau - tab_t[j]) / (tab_t[j + 1] - tab_t[j]);
            }
        }
        coef[k] = ramp * g;
    }
}

/* ------------------------------------------------------------------------------------ */
/* One ensemble SpMM y_s = K_s u_s (the per-step product of PAPER.md:26, 349):           */
/*   y[s][i][c] = sum_{blocks (i,j) in CSR order} sum_{d=0..2} Kval_s[b][c][d] u[s][j][d] */
/* u, y: [n_s][V][3]; Kval: [n_s][nnzb][9].                                               */
/* ------------------------------------------------------------------------------------ */
void orc_spmm(int64_t V, const int64_t* row_ptr, const int32_t* col, int32_t n_s,
              const double* Kval, const double* u, double* y) {
    int64_t nnzb = row_ptr[V];
#pragma omp parallel for schedule(static)
    for (int32_t s = 0; s < n_s; s++) {
        const double* K = Kval + (int64_t)s * nnzb * 9;
        const double* us = u + (int64_t)s * V * 3;
        for (int64_t i = 0; i < V; i++)
            for (int c = 0; c < 3; c++) {
                double acc = 0.0;
                for (int64_t b = row_ptr[i]; b < row_ptr[i + 1]; b++)
                    for (int d = 0; d < 3; d++) acc += K[b * 9 + 3 * c + d] * us[3 * (int64_t)col[b] + d];
                y[(int64_t)s * V * 3 + 3 * i + c] = acc;
            }
    }
}

/* ------------------------------------------------------------------------------------ */
/* n explicit central-difference steps (Eq. 22):   */
/* for each s, each DOF (i,c), at t_n = (step0 + n) dt:                                   */
/*   y = sum_{blocks (i,j)} sum_d Kval_s[i,j][c][d] u_n[j][d]                              */
/*   r = f(t_n)[i][c] - y,        f(t) = sum_k coef_k(t) F_k[i][c]                       */
/*   u_{n+1} = c1 r + c2 u_n - c3 u_{n-1};  fixed DOF (bit c of fixed[i]) => 0.           */
/* u_n, u_nm1: [n_s][V][3], updated in place to (u_{n+step}, u_{n+step-1}).               */
/* Returns -1, or the first step index (absolute) at which a non-finite value appeared.  */
/* ------------------------------------------------------------------------------------ */
int64_t orc_run(int64_t V, const int64_t* row_ptr, const int32_t* col, int32_t n_s,
                const double* Kval, const double* c1, const double* c2, const double* c3,
                const uint8_t* fixed, int32_t K, const double* Fk, int32_t n_tab,
                const double* tab_t, const double* tab_g, double period, double ramp_T,
                double dt, int64_t step0, int64_t nsteps, double* u_n, double* u_nm1) {
    int64_t nnzb = row_ptr[V];
    int64_t bad = -1;
    double* u_np1 = (double*)malloc(sizeof(double) * (size_t)n_s * (size_t)V * 3);
    double coef[16];
    for (int64_t n = 0; n < nsteps; n++) {
        double t = (double)(step0 + n) * dt;
        orc_load_coeffs(t, K, n_tab, tab_t, tab_g, period, ramp_T, coef);
#pragma omp parallel for schedule(static)
        for (int32_t s = 0; s < n_s; s++) {
            const double* Ks = Kval + (int64_t)s * nnzb * 9;
            const double* un = u_n + (int64_t)s * V * 3;
            const double* uo = u_nm1 + (int64_t)s * V * 3;
            double* unew = u_np1 + (int64_t)s * V * 3;
            for (int64_t i = 0; i < V; i++) {
                int64_t node = (int64_t)s * V + i;
                for (int c = 0; c < 3; c++) {
                    double y = 0.0;
                    for (int64_t b = row_ptr[i]; b < row_ptr[i + 1]; b++)
                        for (int d = 0; d < 3; d++) y += Ks[b * 9 + 3 * c + d] * un[3 * (int64_t)col[b] + d];
                    double f = 0.0;
                    for (int32_t k = 0; k < K; k++) f += coef[k] * Fk[((int64_t)k * V + i) * 3 + c];
                    double r = f - y;
                    double v = c1[node] * r + c2[node] * un[3 * i + c] - c3[node] * uo[3 * i + c];
                    if (fixed && ((fixed[i] >> c) & 1)) v = 0.0;
                    unew[3 * i + c] = v;
                }
            }
        }
        for (int64_t t2 = 0; t2 < (int64_t)n_s * V * 3; t2++) {
            if (bad < 0 && !isfinite(u_np1[t2])) bad = step0 + n;
            u_nm1[t2] = u_n[t2];
            u_n[t2] = u_np1[t2];
        }
    }
    free(u_np1);
    return bad;
}

/* ------------------------------------------------------------------------------------ */
/* Node partition and halo maps (the paper's mesh partitions and   */
/* shared-node synchronisation).  Rows are in RCM order.              */
/*   bounds[p] = min { r : P * row_ptr[r] >= p * nnzb }, bounds[0] = 0, bounds[P] = V.    */
/* ------------------------------------------------------------------------------------ */
void orc_partition_bounds(int64_t V, const int64_t* row_ptr, int32_t P, int64_t* bounds) {
    int64_t nnzb = row_ptr[V];
    bounds[0] = 0;
    for (int32_t p = 1; p < P; p++) {
        int64_t r = 0;
        while ((int64_t)P * row_ptr[r] < (int64_t)p * nnzb) r++;
        bounds[p] = r;
    }
    bounds[P] = V;
}

/* ghosts of part p: sorted unique columns j outside [lo, hi) of the rows in [lo, hi). */
int64_t orc_ghosts(int64_t V, const int64_t* row_ptr, const int32_t* col, int64_t lo, int64_t hi,
                   int32_t* ghosts) {
    char* mark = (char*)calloc((size_t)V + 1, 1);
    for (int64_t i = lo; i < hi; i++)
        for (int64_t b = row_ptr[i]; b < row_ptr[i + 1]; b++)
            if (col[b] < lo || col[b] >= hi) mark[col[b]] = 1;
    int64_t n = 0;
    for (int64_t j = 0; j < V; j++)
        if (mark[j]) ghosts[n++] = (int32_t)j;
    free(mark);
    return n;
}

/* ------------------------------------------------------------------------------------ */
/* Stress recovery (Eq. 7-9).  For element e and   */
/* realisation s: local strain eps = B (T u_e) (Eq. 8, constant on the element), stress  */
/* sigma = C(Ebar) eps (Eq. 7, 9) with Ebar the element mean of the nodal E (= the mean  */
/* over the three Gauss points, sigma being linear in E).  frame 0: local shell frame,   */
/* out = (s_xx, s_yy, t_xy, t_xz, t_yz, 0).  frame 1: "cylindrical" frame of PAPER.md:320: */
/* r = the element normal, z = tangent of the centreline at its point closest to the     */
/* element centroid (made orthogonal to r), theta = r x z;                                */
/* out = (s_rr, s_tt, s_zz, s_tz, s_rz, s_rt) of the 3-D tensor [[s_xx t_xy t_xz],        */
/* [t_xy s_yy t_yz], [t_xz t_yz 0]] (eps_zz = 0) rotated from the local     */
/* basis.  centerline: [n_c][3] polyline, or NULL for the z axis.  out: [n_s][F][6].       */
/* ------------------------------------------------------------------------------------ */
static void closest_tangent(const double* c, const double* cl, int32_t n_c, double* tz) {
    if (!cl || n_c < 2) { tz[0] = 0.0; tz[1] = 0.0; tz[2] = 1.0; return; }
    double best = INFINITY;
    for (int32_t k = 0; k + 1 < n_c; k++) {
        const double* A = cl + 3 * k;
        const double* B = cl + 3 * (k + 1);
        double d[3] = {B[0] - A[0], B[1] - A[1], B[2] - A[2]};
        double dd = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
        double t = ((c[0] - A[0]) * d[0] + (c[1] - A[1]) * d[1] + (c[2] - A[2]) * d[2]) / dd;
        if (t < 0.0) t = 0.0;
        if (t > 1.0) t = 1.0;
        double q[3] = {A[0] + t * d[0] - c[0], A[1] + t * d[1] - c[1], A[2] + t * d[2] - c[2]};
        double dist = q[0] * q[0] + q[1] * q[1] + q[2] * q[2];
        if (dist < best) {
            best = dist;
            double nd = sqrt(dd);
            tz[0] = d[0] / nd; tz[1] = d[1] / nd; tz[2] = d[2] / nd;
        }
    }
}

void orc_stress(int64_t V, int64_t F, const double* xyz, const int32_t* tris, int32_t n_s,
                const double* E, const double* u, double nu, double kshear, int32_t frame,
                const double* centerline, int32_t n_c, double* out) {
    for (int64_t e = 0; e < F; e++) {
        const int32_t* t = tris + 3 * e;
        const double* X1 = xyz + 3 * (int64_t)t[0];
        const double* X2 = xyz + 3 * (int64_t)t[1];
        const double* X3 = xyz + 3 * (int64_t)t[2];
        double d21[3], d31[3], n[3], e1[3], e2[3], e3[3];
        for (int c = 0; c < 3; c++) { d21[c] = X2[c] - X1[c]; d31[c] = X3[c] - X1[c]; }
        n[0] = d21[1] * d31[2] - d21[2] * d31[1];
        n[1] = d21[2] * d31[0] - d21[0] * d31[2];
        n[2] = d21[0] * d31[1] - d21[1] * d31[0];
        double nn = sqrt(n[0] * n[0] + n[1] * n[1] + n[2] * n[2]);
        double A = 0.5 * nn;
        double l21 = sqrt(d21[0] * d21[0] + d21[1] * d21[1] + d21[2] * d21[2]);
        for (int c = 0; c < 3; c++) { e1[c] = d21[c] / l21; e3[c] = n[c] / nn; }
        e2[0] = e3[1] * e1[2] - e3[2] * e1[1];
        e2[1] = e3[2] * e1[0] - e3[0] * e1[2];
        e2[2] = e3[0] * e1[1] - e3[1] * e1[0];
        const double* Xs[3] = {X1, X2, X3};
        double x[3], y[3];
        for (int a = 0; a < 3; a++) {
            double d[3] = {Xs[a][0] - X1[0], Xs[a][1] - X1[1], Xs[a][2] - X1[2]};
            x[a] = d[0] * e1[0] + d[1] * e1[1] + d[2] * e1[2];
            y[a] = d[0] * e2[0] + d[1] * e2[1] + d[2] * e2[2];
        }
        double y23 = y[1] - y[2], y31 = y[2] - y[0], y12 = y[0] - y[1];
        double x32 = x[2] - x[1], x13 = x[0] - x[2], x21 = x[1] - x[0];
        double Bm[5][9];
        memset(Bm, 0, sizeof(Bm));
        Bm[0][0] = y23; Bm[0][3] = y31; Bm[0][6] = y12;
        Bm[1][1] = x32; Bm[1][4] = x13; Bm[1][7] = x21;
        Bm[2][0] = x32; Bm[2][1] = y23; Bm[2][3] = x13; Bm[2][4] = y31; Bm[2][6] = x21; Bm[2][7] = y12;
        Bm[3][2] = y23; Bm[3][5] = y31; Bm[3][8] = y12;
        Bm[4][2] = x32; Bm[4][5] = x13; Bm[4][8] = x21;
        /* output basis (rows b_p in global coordinates) */
        double b[3][3];
        if (frame == 1) {
            double cen[3] = {(X1[0] + X2[0] + X3[0]) / 3.0, (X1[1] + X2[1] + X3[1]) / 3.0, (X1[2] + X2[2] + X3[2]) / 3.0};
            double tz[3];
            closest_tangent(cen, centerline, n_c, tz);
            double dz = tz[0] * e3[0] + tz[1] * e3[1] + tz[2] * e3[2];
            double z[3] = {tz[0] - dz * e3[0], tz[1] - dz * e3[1], tz[2] - dz * e3[2]};
            double zn = sqrt(z[0] * z[0] + z[1] * z[1] + z[2] * z[2]);
            for (int c = 0; c < 3; c++) { b[0][c] = e3[c]; b[2][c] = z[c] / zn; }
            b[1][0] = b[0][1] * b[2][2] - b[0][2] * b[2][1];   /* theta = r x z */
            b[1][1] = b[0][2] * b[2][0] - b[0][0] * b[2][2];
            b[1][2] = b[0][0] * b[2][1] - b[0][1] * b[2][0];
        }
        for (int32_t s = 0; s < n_s; s++) {
            const double* us = u + (int64_t)s * V * 3;
            double ul[9];
            for (int a = 0; a < 3; a++) {
                const double* ug = us + 3 * (int64_t)t[a];
                ul[3 * a + 0] = e1[0] * ug[0] + e1[1] * ug[1] + e1[2] * ug[2];
                ul[3 * a + 1] = e2[0] * ug[0] + e2[1] * ug[1] + e2[2] * ug[2];
                ul[3 * a + 2] = e3[0] * ug[0] + e3[1] * ug[1] + e3[2] * ug[2];
            }
            double eps[5];
            for (int r = 0; r < 5; r++) {
                double acc = 0.0;
                for (int k = 0; k < 9; k++) acc += Bm[r][k] * ul[k];
                eps[r] = acc / (2.0 * A);
            }
            double Eb = (E[(int64_t)s * V + t[0]] + E[(int64_t)s * V + t[1]] + E[(int64_t)s * V + t[2]]) / 3.0;
            double pre = Eb / (1.0 - nu * nu);
            double sg[5];
            sg[0] = pre * (eps[0] + nu * eps[1]);
            sg[1] = pre * (nu * eps[0] + eps[1]);
            sg[2] = pre * 0.5 * (1.0 - nu) * eps[2];
            sg[3] = pre * 0.5 * kshear * (1.0 - nu) * eps[3];
            sg[4] = pre * 0.5 * kshear * (1.0 - nu) * eps[4];
            double* o = out + ((int64_t)s * F + e) * 6;
            if (frame == 0) {
                for (int k = 0; k < 5; k++) o[k] = sg[k];
                o[5] = 0.0;
                continue;
            }
            /* S_local -> global -> cylindrical */
            double Sl[3][3] = {{sg[0], sg[2], sg[3]}, {sg[2], sg[1], sg[4]}, {sg[3], sg[4], 0.0}};
            double R[3][3] = {{e1[0], e1[1], e1[2]}, {e2[0], e2[1], e2[2]}, {e3[0], e3[1], e3[2]}};
            double Sg[3][3];
            for (int i = 0; i < 3; i++)
                for (int j = 0; j < 3; j++) {
                    double acc = 0.0;
                    for (int p = 0; p < 3; p++)
                        for (int q = 0; q < 3; q++) acc += R[p][i] * Sl[p][q] * R[q][j];
                    Sg[i][j] = acc;
                }
            double Sc[3][3];
            for (int i = 0; i < 3; i++)
                for (int j = 0; j < 3; j++) {
                    double acc = 0.0;
                    for (int p = 0; p < 3; p++)
                        for (int q = 0; q < 3; q++) acc += b[i][p] * Sg[p][q] * b[j][q];
                    Sc[i][j] = acc;
                }
            o[0] = Sc[0][0]; o[1] = Sc[1][1]; o[2] = Sc[2][2];
            o[3] = Sc[1][2]; o[4] = Sc[0][2]; o[5] = Sc[0][1];
        }
    }
}

/* Thread count of the OpenMP loops over realisations (timing only; results do not depend
 * on it).  Returns the count in effect. */
#ifdef _OPENMP
#include <omp.h>
#endif
int orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
    return omp_get_max_threads();
#else
    (void)n;
    return 1;
#endif
}

/* ------------------------------------------------------------------------------------ */
/* Selective stiffness re-assembly on the updated geometry (SURVEY.md §8(f) N4;         */
/* "the geometry of the vessel lumen is updated at every step by adding    */
/* u_{n+1} ... we provide the option to selectively update the stiffness matrix after a  */
/* prescribed number of iterations").  Realisation s deforms on its own, so             */
/*   Kval_s[i,j] = sum_{e, ascending} alpha_{e,s} K^_e(X + u_n^s)[a(i), b(j)]            */
/* with K^_e(.) = orc_element_khat at the deformed node positions; alpha (material) and  */
/* the lumped mass stay as built ("fixed nodal mass over time").            */
/* ------------------------------------------------------------------------------------ */
int orc_reassemble(int64_t V, int64_t F, const double* xyz, const int32_t* tris, const int64_t* row_ptr,
                   const int32_t* col, double nu, double kshear, int32_t n_s, const double* alpha,
                   const double* u_n, double* Kval) {
    int64_t nnzb = row_ptr[V];
    for (int32_t s = 0; s < n_s; s++) {
        double* K = Kval + (int64_t)s * nnzb * 9;
        const double* us = u_n + (int64_t)s * V * 3;
        for (int64_t t = 0; t < nnzb * 9; t++) K[t] = 0.0;
        for (int64_t e = 0; e < F; e++) {
            double X[9], Kh[81], A;
            for (int a = 0; a < 3; a++)
                for (int c = 0; c < 3; c++) {
                    int64_t node = tris[3 * e + a];
                    X[3 * a + c] = xyz[3 * node + c] + us[3 * node + c];
                }
            orc_element_khat(X, nu, kshear, Kh, &A);
            double al = alpha[(int64_t)s * F + e];
            for (int a = 0; a < 3; a++)
                for (int b = 0; b < 3; b++) {
                    int64_t blk = find_block(row_ptr, col, tris[3 * e + a], tris[3 * e + b]);
                    if (blk < 0) return -1;
                    for (int c = 0; c < 3; c++)
                        for (int d = 0; d < 3; d++) K[blk * 9 + 3 * c + d] += al * Kh[9 * (3 * a + c) + (3 * b + d)];
                }
        }
    }
    return 0;
}
