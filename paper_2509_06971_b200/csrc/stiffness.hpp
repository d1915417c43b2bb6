// stiffness.hpp -- host-side element matrices for the elasticity operator.
//
// unit_cell_stiffness reproduces detail::unit_cell_stiffness
// (state_solver.hpp:149-237) bit for bit (same quadrature, same accumulation
// order, same canonicalisation over the axis-mirror group), because the replica
// kernels apply it in the reference's order.  modal_stiffness() then rotates it
// into the Walsh-Hadamard (corner-parity) basis used by the fast kernels, where
// the 24x24 (3D) / 8x8 (2D) matrix has only 45 / 10 structural nonzeros.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <stdexcept>
#include <vector>

namespace petto_b200 {

// One Gauss point of the 2^dim rule: B-matrix (voigt x dofs) contribution
// weight * B^T D B added into ke, accumulations in the reference's order.
inline std::vector<double> unit_cell_stiffness(int dim, const double h[3], double nu) {
    const int corners = 1 << dim;
    const int ndof = corners * dim;
    const int nv = dim * (dim + 1) / 2;
    const double lam = nu / ((1.0 + nu) * (1.0 - 2.0 * nu));
    const double shear = 1.0 / (2.0 * (1.0 + nu));
    std::vector<double> D(static_cast<size_t>(nv) * nv, 0.0);
    for (int a = 0; a < dim; ++a)
        for (int b = 0; b < dim; ++b) D[a * nv + b] = lam + (a == b ? 2.0 * shear : 0.0);
    for (int s = dim; s < nv; ++s) D[s * nv + s] = shear;
    double vol = 1.0;
    for (int a = 0; a < dim; ++a) vol *= h[a];
    const double w = vol / corners;
    const double gp[2] = {0.5 - 0.5 / std::sqrt(3.0), 0.5 + 0.5 / std::sqrt(3.0)};

    std::vector<double> K(static_cast<size_t>(ndof) * ndof, 0.0);
    std::vector<double> B(static_cast<size_t>(nv) * ndof);
    for (int q = 0; q < corners; ++q) {
        const double xi[3] = {gp[q & 1], gp[(q >> 1) & 1], gp[(q >> 2) & 1]};
        auto grad = [&](int corner, int axis) {  // d N_corner / d x_axis at xi
            double v = 1.0;
            for (int b = 0; b < dim; ++b) {
                const bool hi = (corner >> b) & 1;
                v *= (b == axis) ? (hi ? 1.0 : -1.0) / h[b] : (hi ? xi[b] : 1.0 - xi[b]);
            }
            return v;
        };
        std::fill(B.begin(), B.end(), 0.0);
        for (int m = 0; m < corners; ++m)
            for (int c = 0; c < dim; ++c) {
                const int col = m * dim + c;
                B[c * ndof + col] = grad(m, c);
                int row = dim;  // engineering shears xy, xz, yz
                for (int a = 0; a < dim; ++a)
                    for (int b = a + 1; b < dim; ++b, ++row) {
                        if (c == a) B[row * ndof + col] += grad(m, b);
                        if (c == b) B[row * ndof + col] += grad(m, a);
                    }
            }
        for (int p = 0; p < ndof; ++p)
            for (int r = 0; r < ndof; ++r) {
                double acc = 0.0;
                for (int s = 0; s < nv; ++s) {
                    double db = 0.0;
                    for (int t = 0; t < nv; ++t) db += D[s * nv + t] * B[t * ndof + r];
                    acc += B[s * ndof + p] * db;
                }
                K[p * ndof + r] += w * acc;
            }
    }
    // Canonical representative over {mirror flips} x {transpose}: the smallest
    // (row, col) in lexicographic order among the orbit of each entry, with the
    // sign picked up by the mirrored components.
    std::vector<double> out(K.size());
    for (int p = 0; p < ndof; ++p)
        for (int r = 0; r < ndof; ++r) {
            int bp = p, br = r;
            double sign = 1.0;
            for (int f = 0; f < corners; ++f)
                for (int tr = 0; tr < 2; ++tr) {
                    int pp = ((p / dim) ^ f) * dim + p % dim;
                    int rr = ((r / dim) ^ f) * dim + r % dim;
                    const double sg = (((f >> (p % dim)) & 1) ? -1.0 : 1.0) *
                                      (((f >> (r % dim)) & 1) ? -1.0 : 1.0);
                    if (tr) std::swap(pp, rr);
                    if (pp < bp || (pp == bp && rr < br)) {
                        bp = pp;
                        br = rr;
                        sign = sg;
                    }
                }
            out[p * ndof + r] = sign * K[bp * ndof + br];
        }
    return out;
}

// elasticity_spectral_bound (state_solver.hpp:254-279): power iteration on K_e.
inline double spectral_bound(int dim, const double h[3], double nu, double e_max) {
    const int ndof = (1 << dim) * dim;
    const std::vector<double> K = unit_cell_stiffness(dim, h, nu);
    std::vector<double> v(ndof, 1.0), w(ndof);
    double lmax = 0.0;
    for (int it = 0; it < 200; ++it) {
        double norm = 0.0;
        for (int p = 0; p < ndof; ++p) {
            double acc = 0.0;
            for (int q = 0; q < ndof; ++q) acc += K[p * ndof + q] * v[q];
            w[p] = acc;
            norm += acc * acc;
        }
        norm = std::sqrt(norm);
        if (norm == 0.0) break;
        lmax = norm;
        for (int p = 0; p < ndof; ++p) v[p] = w[p] / norm;
    }
    double vol = 1.0;
    for (int a = 0; a < dim; ++a) vol *= h[a];
    return lmax * e_max * (1 << dim) / vol;
}

// Structural nonzeros of the modal stiffness Khat = T K T / 64 (3D) or / 16 (2D),
// T = kron(H, I_dim), H the corner-parity Walsh-Hadamard matrix.  Each entry is
// (out mode, out comp, in mode, in comp); the fast kernels hard-code this order.
struct ModalEntry {
    int os, oc, is, ic;
};

inline const std::vector<ModalEntry>& modal_pattern(int dim) {
    static const std::vector<ModalEntry> p3 = {
        // linear modes {1 (x), 2 (y), 4 (z)}: normal strains + in-plane shears
        {1, 0, 1, 0}, {1, 0, 2, 1}, {1, 0, 4, 2},
        {1, 1, 1, 1}, {1, 1, 2, 0},
        {1, 2, 1, 2}, {1, 2, 4, 0},
        {2, 0, 1, 1}, {2, 0, 2, 0},
        {2, 1, 1, 0}, {2, 1, 2, 1}, {2, 1, 4, 2},
        {2, 2, 2, 2}, {2, 2, 4, 1},
        {4, 0, 1, 2}, {4, 0, 4, 0},
        {4, 1, 2, 2}, {4, 1, 4, 1},
        {4, 2, 1, 0}, {4, 2, 2, 1}, {4, 2, 4, 2},
        // bilinear modes {3 (xy), 5 (xz), 6 (yz)}
        {3, 0, 3, 0}, {3, 0, 6, 2},
        {3, 1, 3, 1}, {3, 1, 5, 2},
        {3, 2, 3, 2}, {3, 2, 5, 1}, {3, 2, 6, 0},
        {5, 0, 5, 0}, {5, 0, 6, 1},
        {5, 1, 3, 2}, {5, 1, 5, 1}, {5, 1, 6, 0},
        {5, 2, 3, 1}, {5, 2, 5, 2},
        {6, 0, 3, 2}, {6, 0, 5, 1}, {6, 0, 6, 0},
        {6, 1, 5, 0}, {6, 1, 6, 1},
        {6, 2, 3, 0}, {6, 2, 6, 2},
        // trilinear mode 7
        {7, 0, 7, 0}, {7, 1, 7, 1}, {7, 2, 7, 2},
    };
    static const std::vector<ModalEntry> p2 = {
        {1, 0, 1, 0}, {1, 0, 2, 1}, {1, 1, 1, 1}, {1, 1, 2, 0},
        {2, 0, 1, 1}, {2, 0, 2, 0}, {2, 1, 1, 0}, {2, 1, 2, 1},
        {3, 0, 3, 0}, {3, 1, 3, 1},
    };
    return dim == 3 ? p3 : p2;
}

// Khat values in modal_pattern order.  Throws if K has weight outside the
// pattern (would mean the element is not the axis-aligned isotropic one).
inline std::vector<double> modal_stiffness(int dim, const std::vector<double>& K) {
    const int corners = 1 << dim;
    const int ndof = corners * dim;
    auto H = [](int s, int m) { return (__builtin_popcount(s & m) & 1) ? -1.0L : 1.0L; };
    std::vector<long double> Kh(static_cast<size_t>(ndof) * ndof, 0.0L);
    long double kmax = 0.0L;
    for (int s = 0; s < corners; ++s)
        for (int c = 0; c < dim; ++c)
            for (int t = 0; t < corners; ++t)
                for (int e = 0; e < dim; ++e) {
                    long double acc = 0.0L;
                    for (int m = 0; m < corners; ++m)
                        for (int n = 0; n < corners; ++n)
                            acc += H(s, m) * (long double)K[(m * dim + c) * ndof + n * dim + e] * H(t, n);
                    acc /= (long double)(corners * corners);
                    Kh[(s * dim + c) * ndof + t * dim + e] = acc;
                    if (fabsl(acc) > kmax) kmax = fabsl(acc);
                }
    const auto& pat = modal_pattern(dim);
    std::vector<char> used(Kh.size(), 0);
    std::vector<double> out;
    for (const ModalEntry& e : pat) {
        const size_t idx = static_cast<size_t>(e.os * dim + e.oc) * ndof + e.is * dim + e.ic;
        used[idx] = 1;
        out.push_back(static_cast<double>(Kh[idx]));
    }
    for (size_t i = 0; i < Kh.size(); ++i)
        if (!used[i] && fabsl(Kh[i]) > 1e-12L * kmax)
            throw std::runtime_error("modal stiffness: entry outside the structural pattern");
    return out;
}

}  // namespace petto_b200
