// host_setup.cpp -- one-time host setup (see host_setup.hpp).  C++17, no CUDA.
#include "host_setup.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <numeric>

namespace ens {

namespace {

inline std::array<double, 3> sub(const double* a, const double* b) {
    return {a[0] - b[0], a[1] - b[1], a[2] - b[2]};
}
inline std::array<double, 3> cross(const std::array<double, 3>& a, const std::array<double, 3>& b) {
    return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
inline double dot(const std::array<double, 3>& a, const std::array<double, 3>& b) {
    return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}
inline double norm(const std::array<double, 3>& a) { return std::sqrt(dot(a, a)); }

}  // namespace

// ------------------------------------------------------------------------------------
// Mesh validation.  Degenerate: A_e <= 1e-12 * (sum of squared edge lengths)
// (the scale-free form of "A_e > 0").
// ------------------------------------------------------------------------------------
int validate_mesh(const MeshView& m, int64_t* bad) {
    *bad = -1;
    for (int64_t e = 0; e < m.F; ++e) {
        const int32_t* t = m.tris + 3 * e;
        for (int a = 0; a < 3; ++a)
            if (t[a] < 0 || t[a] >= m.V) { *bad = e; return 1; }
        if (t[0] == t[1] || t[1] == t[2] || t[0] == t[2]) { *bad = e; return 2; }
        const double* P = m.xyz + 3 * int64_t(t[0]);
        const double* Q = m.xyz + 3 * int64_t(t[1]);
        const double* R = m.xyz + 3 * int64_t(t[2]);
        auto pq = sub(Q, P), qr = sub(R, Q), rp = sub(P, R);
        double l2 = 0.0;
        for (int c = 0; c < 3; ++c) l2 += pq[c] * pq[c] + qr[c] * qr[c] + rp[c] * rp[c];
        double area = 0.5 * norm(cross(sub(Q, P), sub(R, P)));
        if (!(area > 1e-12 * l2)) { *bad = e; return 3; }
    }
    std::vector<uint64_t> keys;
    keys.reserve(size_t(3 * m.F));
    for (int64_t e = 0; e < m.F; ++e)
        for (int a = 0; a < 3; ++a) {
            uint64_t p = uint32_t(m.tris[3 * e + a]), q = uint32_t(m.tris[3 * e + (a + 1) % 3]);
            keys.push_back(p < q ? (p << 32 | q) : (q << 32 | p));
        }
    std::sort(keys.begin(), keys.end());
    for (size_t k = 0; k + 2 < keys.size(); ++k)
        if (keys[k] == keys[k + 2]) { *bad = int64_t(keys[k] >> 32); return 4; }
    // every node must lie in a triangle: its lumped mass rho sum A_e zeta/3
    // is the divisor of c1, so an unreferenced node would turn the first step into NaN
    std::vector<char> used(size_t(m.V), 0);
    for (int64_t k = 0; k < 3 * m.F; ++k) used[size_t(m.tris[k])] = 1;
    for (int64_t i = 0; i < m.V; ++i)
        if (!used[size_t(i)]) { *bad = i; return 5; }
    return 0;
}

// ------------------------------------------------------------------------------------
// Edge graph + RCM + CSR.
// ------------------------------------------------------------------------------------
void edge_graph(const MeshView& m, std::vector<int64_t>& ptr, std::vector<int32_t>& adj) {
    std::vector<uint64_t> keys;
    keys.reserve(size_t(6 * m.F));
    for (int64_t e = 0; e < m.F; ++e) {
        const int32_t* t = m.tris + 3 * e;
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b)
                if (a != b) keys.push_back(uint64_t(uint32_t(t[a])) << 32 | uint32_t(t[b]));
    }
    std::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    ptr.assign(size_t(m.V + 1), 0);
    adj.resize(keys.size());
    for (size_t k = 0; k < keys.size(); ++k) {
        ptr[size_t(keys[k] >> 32) + 1]++;
        adj[k] = int32_t(keys[k] & 0xffffffffu);
    }
    std::partial_sum(ptr.begin(), ptr.end(), ptr.begin());
}

namespace {

struct Bfs {
    std::vector<int32_t> level, order;
    int32_t ecc = 0;
    // level structure rooted at r; order = BFS order (component only)
    void run(const std::vector<int64_t>& ptr, const std::vector<int32_t>& adj, int32_t r) {
        for (int32_t v : order) level[size_t(v)] = -1;
        order.clear();
        order.push_back(r);
        level[size_t(r)] = 0;
        ecc = 0;
        for (size_t h = 0; h < order.size(); ++h) {
            int32_t v = order[h];
            for (int64_t k = ptr[size_t(v)]; k < ptr[size_t(v) + 1]; ++k) {
                int32_t w = adj[size_t(k)];
                if (level[size_t(w)] < 0) {
                    level[size_t(w)] = level[size_t(v)] + 1;
                    ecc = std::max(ecc, level[size_t(w)]);
                    order.push_back(w);
                }
            }
        }
    }
};

}  // namespace

std::vector<int32_t> rcm_order(int64_t V, const std::vector<int64_t>& ptr, const std::vector<int32_t>& adj) {
    std::vector<int64_t> deg(static_cast<size_t>(V));
    for (int64_t i = 0; i < V; ++i) deg[size_t(i)] = ptr[size_t(i) + 1] - ptr[size_t(i)];
    auto less_key = [&](int32_t a, int32_t b) {
        return deg[size_t(a)] != deg[size_t(b)] ? deg[size_t(a)] < deg[size_t(b)] : a < b;
    };
    Bfs bfs;
    bfs.level.assign(size_t(V), -1);
    std::vector<char> placed(size_t(V), 0);
    std::vector<int32_t> cm;
    cm.reserve(size_t(V));
    std::vector<int32_t> nb;
    for (int32_t c0 = 0; c0 < V; ++c0) {
        if (placed[size_t(c0)]) continue;
        bfs.run(ptr, adj, c0);                                   // the component of c0
        int32_t r = *std::min_element(bfs.order.begin(), bfs.order.end(), less_key);
        bfs.run(ptr, adj, r);
        for (;;) {                                               // George-Liu
            int32_t ecc_r = bfs.ecc, x = -1;
            for (int32_t v : bfs.order)
                if (bfs.level[size_t(v)] == ecc_r && (x < 0 || less_key(v, x))) x = v;
            bfs.run(ptr, adj, x);
            if (bfs.ecc > ecc_r) {
                r = x;
            } else {
                bfs.run(ptr, adj, r);                            // restore r's levels
                break;
            }
        }
        size_t head = cm.size();
        cm.push_back(r);
        placed[size_t(r)] = 1;
        while (head < cm.size()) {
            int32_t v = cm[head++];
            nb.clear();
            for (int64_t k = ptr[size_t(v)]; k < ptr[size_t(v) + 1]; ++k)
                if (!placed[size_t(adj[size_t(k)])]) nb.push_back(adj[size_t(k)]);
            std::sort(nb.begin(), nb.end(), less_key);
            for (int32_t w : nb) {
                placed[size_t(w)] = 1;
                cm.push_back(w);
            }
        }
    }
    std::reverse(cm.begin(), cm.end());
    return cm;
}

Pattern build_pattern(const MeshView& m) {
    std::vector<int64_t> ptr;
    std::vector<int32_t> adj;
    edge_graph(m, ptr, adj);
    Pattern p;
    p.perm = rcm_order(m.V, ptr, adj);
    p.iperm.assign(size_t(m.V), 0);
    for (int64_t i = 0; i < m.V; ++i) p.iperm[size_t(p.perm[size_t(i)])] = int32_t(i);
    p.row_ptr.assign(size_t(m.V + 1), 0);
    p.col.reserve(size_t(m.V) + adj.size());
    for (int64_t i = 0; i < m.V; ++i) {
        int32_t old = p.perm[size_t(i)];
        size_t start = p.col.size();
        p.col.push_back(int32_t(i));
        for (int64_t k = ptr[size_t(old)]; k < ptr[size_t(old) + 1]; ++k) p.col.push_back(p.iperm[size_t(adj[size_t(k)])]);
        std::sort(p.col.begin() + int64_t(start), p.col.end());
        p.row_ptr[size_t(i) + 1] = int64_t(p.col.size());
        for (size_t k = start; k < p.col.size(); ++k)
            p.bandwidth = std::max<int32_t>(p.bandwidth, std::abs(p.col[k] - int32_t(i)));
    }
    return p;
}

// ------------------------------------------------------------------------------------
// Element stiffness (Eqs. 7-10) in closed form.  With the shape
// function gradients dN_a/dx = b_a / 2A, dN_a/dy = c_a / 2A (b = y23, y31, y12;
// c = x32, x13, x21, Eq. 8), pre = 1/(1-nu^2), g = (1-nu)/2:
//   membrane  k[ax][bx] = q (b_a b_b + g c_a c_b)    k[ax][by] = q (nu b_a c_b + g c_a b_b)
//             k[ay][bx] = q (nu c_a b_b + g b_a c_b) k[ay][by] = q (c_a c_b + g b_a b_b)
//   shear     k[az][bz] = q g k_s (b_a b_b + c_a c_b),          q = pre / (4 A)
// then K^_ab = R^T k_ab R with R = [e1; e2; e3] (rows), e1 along X1->X2, e3 the normal.
// ------------------------------------------------------------------------------------
void element_stiffness(const double* X1, const double* X2, const double* X3, double nu,
                       double k_shear, double* Khat, double* area) {
    auto d21 = sub(X2, X1), d31 = sub(X3, X1);
    auto n = cross(d21, d31);
    double nn = norm(n), A = 0.5 * nn, l = norm(d21);
    std::array<double, 3> e1{d21[0] / l, d21[1] / l, d21[2] / l};
    std::array<double, 3> e3{n[0] / nn, n[1] / nn, n[2] / nn};
    auto e2 = cross(e3, e1);
    const double* X[3] = {X1, X2, X3};
    double x[3], y[3];
    for (int a = 0; a < 3; ++a) {
        auto d = sub(X[a], X1);
        x[a] = dot(d, e1);
        y[a] = dot(d, e2);
    }
    double b[3] = {y[1] - y[2], y[2] - y[0], y[0] - y[1]};
    double c[3] = {x[2] - x[1], x[0] - x[2], x[1] - x[0]};
    double pre = 1.0 / (1.0 - nu * nu), g = 0.5 * (1.0 - nu), q = pre / (4.0 * A);
    double R[3][3] = {{e1[0], e1[1], e1[2]}, {e2[0], e2[1], e2[2]}, {e3[0], e3[1], e3[2]}};
    for (int a = 0; a < 3; ++a)
        for (int bb = 0; bb < 3; ++bb) {
            double kl[3][3] = {
                {q * (b[a] * b[bb] + g * c[a] * c[bb]), q * (nu * b[a] * c[bb] + g * c[a] * b[bb]), 0.0},
                {q * (nu * c[a] * b[bb] + g * b[a] * c[bb]), q * (c[a] * c[bb] + g * b[a] * b[bb]), 0.0},
                {0.0, 0.0, q * g * k_shear * (b[a] * b[bb] + c[a] * c[bb])}};
            for (int i = 0; i < 3; ++i)
                for (int j = 0; j < 3; ++j) {
                    double s = 0.0;
                    for (int p = 0; p < 3; ++p)
                        for (int r = 0; r < 3; ++r) s += R[p][i] * kl[p][r] * R[r][j];
                    Khat[9 * (3 * a + i) + (3 * bb + j)] = s;
                }
        }
    for (int i = 0; i < 9; ++i)          // exact symmetry: mirror the upper triangle
        for (int j = i + 1; j < 9; ++j) Khat[9 * j + i] = Khat[9 * i + j];
    *area = A;
}

// ------------------------------------------------------------------------------------
// Stress recovery operators.  With b_a, c_a as in element_stiffness:
// eps_xx = sum b_a ux_a / 2A, eps_yy = sum c_a uy_a / 2A, gamma_xy = sum (c_a ux_a + b_a uy_a)
// / 2A, gamma_xz = sum b_a uz_a / 2A, gamma_yz = sum c_a uz_a / 2A (Eq. 8), u_local = R u.
// ------------------------------------------------------------------------------------
void element_strain_operator(const double* X1, const double* X2, const double* X3, double* G, double* R) {
    auto d21 = sub(X2, X1), d31 = sub(X3, X1);
    auto n = cross(d21, d31);
    const double nn = norm(n), A = 0.5 * nn, l = norm(d21);
    std::array<double, 3> e1{d21[0] / l, d21[1] / l, d21[2] / l};
    std::array<double, 3> e3{n[0] / nn, n[1] / nn, n[2] / nn};
    auto e2 = cross(e3, e1);
    const double* X[3] = {X1, X2, X3};
    double x[3], y[3];
    for (int a = 0; a < 3; ++a) {
        auto d = sub(X[a], X1);
        x[a] = dot(d, e1);
        y[a] = dot(d, e2);
    }
    const double b[3] = {y[1] - y[2], y[2] - y[0], y[0] - y[1]};
    const double c[3] = {x[2] - x[1], x[0] - x[2], x[1] - x[0]};
    const double f = 1.0 / (2.0 * A);
    const std::array<double, 3>* E[3] = {&e1, &e2, &e3};
    for (int a = 0; a < 3; ++a)
        for (int d = 0; d < 3; ++d) {              // global component d of node a
            const double ex = e1[d], ey = e2[d], ez = e3[d];
            G[0 * 9 + 3 * a + d] = f * b[a] * ex;
            G[1 * 9 + 3 * a + d] = f * c[a] * ey;
            G[2 * 9 + 3 * a + d] = f * (c[a] * ex + b[a] * ey);
            G[3 * 9 + 3 * a + d] = f * b[a] * ez;
            G[4 * 9 + 3 * a + d] = f * c[a] * ez;
        }
    for (int r = 0; r < 3; ++r)
        for (int d = 0; d < 3; ++d) R[3 * r + d] = (*E[r])[d];
}

void stress_frame(const double* centroid, const double* R, int32_t frame, const double* centerline,
                  int32_t n_c, double* M) {
    if (frame == 0) {
        for (int k = 0; k < 9; ++k) M[k] = (k % 4 == 0) ? 1.0 : 0.0;
        return;
    }
    std::array<double, 3> tz{0.0, 0.0, 1.0};
    if (centerline && n_c >= 2) {
        double best = INFINITY;
        for (int32_t k = 0; k + 1 < n_c; ++k) {
            const double* P = centerline + 3 * k;
            const double* Q = centerline + 3 * (k + 1);
            auto d = sub(Q, P);
            const double dd = dot(d, d);
            double t = dot(sub(centroid, P), d) / dd;
            t = std::min(1.0, std::max(0.0, t));
            const std::array<double, 3> q{P[0] + t * d[0] - centroid[0], P[1] + t * d[1] - centroid[1],
                                          P[2] + t * d[2] - centroid[2]};
            const double dist = dot(q, q);
            if (dist < best) {
                best = dist;
                const double nd = std::sqrt(dd);
                tz = {d[0] / nd, d[1] / nd, d[2] / nd};
            }
        }
    }
    const std::array<double, 3> r{R[6], R[7], R[8]};
    const double rz = dot(tz, r);
    std::array<double, 3> z{tz[0] - rz * r[0], tz[1] - rz * r[1], tz[2] - rz * r[2]};
    const double zn = norm(z);
    z = {z[0] / zn, z[1] / zn, z[2] / zn};
    const auto th = cross(r, z);
    const std::array<double, 3>* bas[3] = {&r, &th, &z};
    for (int p = 0; p < 3; ++p)                     // M = b R^T: M[p][q] = b_p . e_q
        for (int q = 0; q < 3; ++q)
            M[3 * p + q] = (*bas[p])[0] * R[3 * q] + (*bas[p])[1] * R[3 * q + 1] + (*bas[p])[2] * R[3 * q + 2];
}

// ------------------------------------------------------------------------------------
// alpha_{e,s} = sum_g w_g E_g zeta_g (Eq. 10 with the 3-point rule)
// = (1/12) [ (sum_a E_a)(sum_a zeta_a) + sum_a E_a zeta_a ] exactly for P1 fields.
// m_{i,s} = rho sum_{e ni i} A_e zetabar_{e,s} / 3 (lumped).
// ------------------------------------------------------------------------------------
void materials(const MeshView& m, int32_t n_s, const double* E, const double* h, double rho,
               double* alpha, double* mass) {
    std::vector<double> area(size_t(m.F));
    for (int64_t e = 0; e < m.F; ++e) {
        const int32_t* t = m.tris + 3 * e;
        const double* P = m.xyz + 3 * int64_t(t[0]);
        area[size_t(e)] = 0.5 * norm(cross(sub(m.xyz + 3 * int64_t(t[1]), P), sub(m.xyz + 3 * int64_t(t[2]), P)));
    }
    for (int32_t s = 0; s < n_s; ++s) {
        const double* Es = E + int64_t(s) * m.V;
        const double* hs = h + int64_t(s) * m.V;
        double* ms = mass + int64_t(s) * m.V;
        std::fill(ms, ms + m.V, 0.0);
        for (int64_t e = 0; e < m.F; ++e) {
            const int32_t* t = m.tris + 3 * e;
            double E0 = Es[t[0]], E1 = Es[t[1]], E2 = Es[t[2]];
            double h0 = hs[t[0]], h1 = hs[t[1]], h2 = hs[t[2]];
            alpha[int64_t(s) * m.F + e] = ((E0 + E1 + E2) * (h0 + h1 + h2) + (E0 * h0 + E1 * h1 + E2 * h2)) / 12.0;
            double me = rho * area[size_t(e)] * ((h0 + h1 + h2) / 3.0) / 3.0;
            ms[t[0]] += me;
            ms[t[1]] += me;
            ms[t[2]] += me;
        }
    }
}

// CFL: safety * min_e (4 A_e / perimeter_e) / sqrt(E_max / rho), E_max
// the largest Gauss-point E (interior 3-point rule) over elements and realisations.
double cfl_dt(const MeshView& m, int32_t n_s, const double* E, double rho, double safety) {
    double dmin = INFINITY, Emax = 0.0;
    for (int64_t e = 0; e < m.F; ++e) {
        const int32_t* t = m.tris + 3 * e;
        const double* P[3] = {m.xyz + 3 * int64_t(t[0]), m.xyz + 3 * int64_t(t[1]), m.xyz + 3 * int64_t(t[2])};
        double per = norm(sub(P[1], P[0])) + norm(sub(P[2], P[1])) + norm(sub(P[0], P[2]));
        double A = 0.5 * norm(cross(sub(P[1], P[0]), sub(P[2], P[0])));
        dmin = std::min(dmin, 4.0 * A / per);
        for (int32_t s = 0; s < n_s; ++s) {
            const double* Es = E + int64_t(s) * m.V;
            double a = Es[t[0]], b = Es[t[1]], c = Es[t[2]];
            // Gauss points (2/3,1/6,1/6) and permutations: the max is at the largest node
            double hi = std::max(a, std::max(b, c));
            double g = (2.0 / 3.0) * hi + (1.0 / 6.0) * (a + b + c - hi);
            Emax = std::max(Emax, g);
        }
    }
    return safety * dmin / std::sqrt(Emax / rho);
}

// ------------------------------------------------------------------------------------
// Fans for the matrix-free gather.  Element e = (t0, t1, t2) seen from its local node a
// has the other nodes o1 = t[a+1], o2 = t[a+2] (cyclic, counter-clockwise about the
// outward normal).  On a consistently oriented manifold the next element counter-
// clockwise around the node has o1' = o2, so incidences chain by o2 -> o1.  Chains start
// at an incidence whose o1 is no other incidence's o2 (open fan), else at the smallest
// element; any mesh (even inconsistently oriented) is handled: a chain that cannot be
// continued simply restarts.
// ------------------------------------------------------------------------------------
Fans build_fans(const MeshView& m, const std::vector<int32_t>& iperm, const std::vector<double>& Khat) {
    const int64_t V = m.V, F = m.F;
    Fans f;
    f.ptr.assign(size_t(V) + 1, 0);
    for (int64_t e = 0; e < F; ++e)
        for (int a = 0; a < 3; ++a) f.ptr[size_t(iperm[size_t(m.tris[3 * e + a])]) + 1]++;
    std::partial_sum(f.ptr.begin(), f.ptr.end(), f.ptr.begin());
    // raw incidences per row, ascending element
    std::vector<std::pair<int32_t, int32_t>> raw(size_t(3 * F));   // (e, a)
    std::vector<int32_t> fill(f.ptr.begin(), f.ptr.end() - 1);
    for (int64_t e = 0; e < F; ++e)
        for (int a = 0; a < 3; ++a) raw[size_t(fill[size_t(iperm[size_t(m.tris[3 * e + a])])]++)] = {int32_t(e), a};
    f.rec.resize(size_t(3 * F));
    f.Krow.assign(size_t(3 * F) * 28, 0.0);
    std::vector<char> used;
    for (int64_t i = 0; i < V; ++i) {
        const int32_t lo = f.ptr[size_t(i)], hi = f.ptr[size_t(i) + 1], n = hi - lo;
        auto other = [&](int32_t k, int s) {          // s = 1 -> o1, 2 -> o2 (RCM ids)
            auto [e, a] = raw[size_t(lo + k)];
            return iperm[size_t(m.tris[3 * int64_t(e) + (a + s) % 3])];
        };
        used.assign(size_t(n), 0);
        int32_t out = lo;
        for (int32_t placed = 0; placed < n;) {
            // chain start: an unused incidence whose o1 is not the o2 of another unused one
            int32_t start = -1;
            for (int32_t k = 0; k < n && start < 0; ++k) {
                if (used[size_t(k)]) continue;
                bool has_pred = false;
                for (int32_t q = 0; q < n; ++q)
                    if (q != k && !used[size_t(q)] && other(q, 2) == other(k, 1)) { has_pred = true; break; }
                if (!has_pred) start = k;
            }
            if (start < 0)
                for (int32_t k = 0; k < n; ++k)
                    if (!used[size_t(k)]) { start = k; break; }
            int32_t cur = start;
            bool first = true;
            while (cur >= 0) {
                used[size_t(cur)] = 1;
                ++placed;
                auto [e, a] = raw[size_t(lo + cur)];
                FanRec& r = f.rec[size_t(out)];
                r.e = e;
                r.n_prev = other(cur, 1);
                r.n_next = other(cur, 2);
                r.restart = first ? 1 : 0;
                const int loc[3] = {a, (a + 1) % 3, (a + 2) % 3};
                double* K = f.Krow.data() + size_t(out) * 28;
                for (int c = 0; c < 3; ++c)
                    for (int b = 0; b < 3; ++b)
                        for (int d = 0; d < 3; ++d)
                            K[9 * c + 3 * b + d] = Khat[size_t(e) * 81 + size_t(9 * (3 * a + c) + 3 * loc[b] + d)];
                ++out;
                first = false;
                int32_t nxt = -1;
                for (int32_t q = 0; q < n; ++q)
                    if (!used[size_t(q)] && other(q, 1) == r.n_next) { nxt = q; break; }
                cur = nxt;
            }
        }
    }
    return f;
}

// ------------------------------------------------------------------------------------
// SPDE/GMRF system (see host_setup.hpp).
// ------------------------------------------------------------------------------------
void gmrf_system(const MeshView& m, const Pattern& pat, double kappa, std::vector<double>& val,
                 std::vector<double>& diag, std::vector<double>& lumped) {
    const int64_t V = m.V;
    val.assign(pat.col.size(), 0.0);
    lumped.assign(size_t(V), 0.0);
    for (int64_t e = 0; e < m.F; ++e) {
        const int32_t* t = m.tris + 3 * e;
        const double* X[3] = {m.xyz + 3 * int64_t(t[0]), m.xyz + 3 * int64_t(t[1]), m.xyz + 3 * int64_t(t[2])};
        const double A = 0.5 * norm(cross(sub(X[1], X[0]), sub(X[2], X[0])));
        const std::array<double, 3> ed[3] = {sub(X[2], X[1]), sub(X[0], X[2]), sub(X[1], X[0])};
        for (int a = 0; a < 3; ++a) {
            const int32_t i = pat.iperm[size_t(t[a])];
            lumped[size_t(i)] += A / 3.0;
            for (int b = 0; b < 3; ++b) {
                const int32_t j = pat.iperm[size_t(t[b])];
                auto first = pat.col.begin() + pat.row_ptr[size_t(i)];
                auto last = pat.col.begin() + pat.row_ptr[size_t(i) + 1];
                const int64_t k = int64_t(std::lower_bound(first, last, j) - pat.col.begin());
                val[size_t(k)] += dot(ed[a], ed[b]) / (4.0 * A);
            }
        }
    }
    diag.assign(size_t(V), 0.0);
    for (int64_t i = 0; i < V; ++i)
        for (int64_t k = pat.row_ptr[size_t(i)]; k < pat.row_ptr[size_t(i) + 1]; ++k)
            if (pat.col[size_t(k)] == i) {
                val[size_t(k)] += kappa * kappa * lumped[size_t(i)];
                diag[size_t(i)] = val[size_t(k)];
            }
}

// ------------------------------------------------------------------------------------
// Partition: bounds[p] = min { r : P row_ptr[r] >= p nnzb }.
// ------------------------------------------------------------------------------------
std::vector<int64_t> partition_bounds(const std::vector<int64_t>& row_ptr, int32_t P) {
    int64_t V = int64_t(row_ptr.size()) - 1, nnzb = row_ptr.back();
    std::vector<int64_t> b(size_t(P) + 1, 0);
    for (int32_t p = 1; p < P; ++p) {
        // first r with P * row_ptr[r] >= p * nnzb (row_ptr is non-decreasing)
        auto it = std::partition_point(row_ptr.begin(), row_ptr.end(),
                                       [&](int64_t x) { return int64_t(P) * x < int64_t(p) * nnzb; });
        b[size_t(p)] = int64_t(it - row_ptr.begin());
    }
    b[size_t(P)] = V;
    return b;
}

std::vector<int32_t> ghost_rows(const std::vector<int64_t>& row_ptr, const std::vector<int32_t>& col,
                                int64_t lo, int64_t hi) {
    std::vector<int32_t> g;
    for (int64_t i = lo; i < hi; ++i)
        for (int64_t k = row_ptr[size_t(i)]; k < row_ptr[size_t(i) + 1]; ++k)
            if (col[size_t(k)] < lo || col[size_t(k)] >= hi) g.push_back(col[size_t(k)]);
    std::sort(g.begin(), g.end());
    g.erase(std::unique(g.begin(), g.end()), g.end());
    return g;
}

std::vector<PartPlan> halo_plan(const std::vector<int64_t>& row_ptr, const std::vector<int32_t>& col, int32_t P) {
    const std::vector<int64_t> b = partition_bounds(row_ptr, P);
    std::vector<PartPlan> plans(static_cast<size_t>(P));
    for (int32_t p = 0; p < P; ++p) {
        PartPlan& pl = plans[size_t(p)];
        pl.p = p;
        pl.lo = b[size_t(p)];
        pl.hi = b[size_t(p) + 1];
        pl.ghosts = ghost_rows(row_ptr, col, pl.lo, pl.hi);
        int64_t last_lo = -1, first_hi = pl.n_own();
        for (int64_t i = pl.lo; i < pl.hi; ++i)
            for (int64_t k = row_ptr[size_t(i)]; k < row_ptr[size_t(i) + 1]; ++k) {
                if (col[size_t(k)] < pl.lo) last_lo = std::max(last_lo, i - pl.lo);
                if (col[size_t(k)] >= pl.hi) first_hi = std::min(first_hi, i - pl.lo);
            }
        pl.b_lo = last_lo + 1;
        pl.b_hi = pl.n_own() - first_hi;
        if (pl.b_lo + pl.b_hi > pl.n_own()) { pl.b_lo = pl.n_own(); pl.b_hi = 0; }
    }
    for (int32_t p = 0; p < P; ++p) {
        PartPlan& pl = plans[size_t(p)];
        for (int32_t q = 0; q < P; ++q) {
            if (q == p) continue;
            const PartPlan& ql = plans[size_t(q)];
            PartPlan::Peer pe;
            pe.q = q;
            pe.send_off = int64_t(pl.send_rows.size());
            for (int32_t g : ql.ghosts)                       // my rows that q needs, ascending
                if (g >= pl.lo && g < pl.hi) pl.send_rows.push_back(int32_t(g - pl.lo));
            pe.send_n = int64_t(pl.send_rows.size()) - pe.send_off;
            auto first = std::lower_bound(pl.ghosts.begin(), pl.ghosts.end(), int32_t(ql.lo));
            auto last = std::lower_bound(pl.ghosts.begin(), pl.ghosts.end(), int32_t(ql.hi));
            pe.recv_row = pl.n_own() + int64_t(first - pl.ghosts.begin());
            pe.recv_n = int64_t(last - first);
            if (pe.send_n || pe.recv_n) pl.peers.push_back(pe);
        }
    }
    return plans;
}

}  // namespace ens
