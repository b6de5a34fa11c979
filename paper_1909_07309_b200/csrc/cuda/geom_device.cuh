// Device helpers shared by the physical assembly / stencil kernels (physical.cu) and the space-time
// RHS / error-norm kernels (spacetime.cu): catalog coefficient fields, uniform-knot B-spline
// evaluation (bspline.cpp:14-130) and the spline geometry map with its Jacobian (geometry.cpp:41-97).
#pragma once

#include "physical.cuh"

namespace stiga {
namespace gpu {
namespace geomdev {

constexpr double kPi = 3.14159265358979323846;
constexpr int kMaxP = 8;

__device__ __forceinline__ double field(int kind, const double* x) {
    switch (kind) {
        case kFieldSeparableNu: return 50.5 + 49.5 * x[1] / hypot(x[0], x[1]);                       // problems.cpp:224-227
        case kFieldDeformedKappa: return 1.0 + 0.5 * sin(2.0 * kPi * x[0]) * cos(2.0 * kPi * x[1]);   // BASELINE c4
        case kFieldDeformedC: return 1.0 + 0.25 * x[2];                                               // BASELINE c4
        default: return 1.0;
    }
}

// Knot t_i of the uniform open knot vector of degree p with ne elements.
__device__ __forceinline__ double uknot(int i, int p, int ne) {
    const int k = i - p;
    return k <= 0 ? 0.0 : (k >= ne ? 1.0 : static_cast<double>(k) / ne);
}

// Cox-De Boor values of the deg+1 functions non-zero on span k (bspline.cpp:14-29).
__device__ __forceinline__ void cox(int k, int deg, int p, int ne, double x, double* N) {
    double left[kMaxP + 1], right[kMaxP + 1];
    N[0] = 1.0;
    for (int j = 1; j <= deg; ++j) {
        left[j] = x - uknot(k + 1 - j, p, ne);
        right[j] = uknot(k + j, p, ne) - x;
        double saved = 0.0;
        for (int r = 0; r < j; ++r) {
            const double den = right[r + 1] + left[j - r];
            const double temp = den != 0.0 ? N[r] / den : 0.0;
            N[r] = saved + right[r + 1] * temp;
            saved = left[j - r] * temp;
        }
        N[j] = saved;
    }
}

// Values and first derivatives of the p+1 B-splines at x (bspline.cpp:100-130); returns first index.
__device__ __forceinline__ int basis(double x, int p, int ne, double* val, double* der) {
    int e = static_cast<int>(floor(x * ne));
    e = min(max(e, 0), ne - 1);
    const int k = e + p;
    cox(k, p, p, ne, x, val);
    double low[kMaxP + 1];
    if (p == 1) low[0] = 1.0;
    else cox(k, p - 1, p, ne, x, low);
    for (int r = 0; r <= p; ++r) {
        const int i = k - p + r;
        double dv = 0.0;
        if (r > 0) {
            const double den = uknot(i + p, p, ne) - uknot(i, p, ne);
            if (den != 0.0) dv += low[r - 1] / den;
        }
        if (r < p) {
            const double den = uknot(i + p + 1, p, ne) - uknot(i + 1, p, ne);
            if (den != 0.0) dv -= low[r] / den;
        }
        der[r] = p * dv;
    }
    return k - p;
}

// F(eta) and J = dF/deta (geometry.cpp:41-97) of the uniform-knot spline map.
template <int D>
__device__ void geometry_eval(const PhysicalDesc& g, const double* eta, double* x, double* J) {
    double val[D][kMaxP + 1], der[D][kMaxP + 1];
    int first[D];
    for (int l = 0; l < D; ++l) first[l] = basis(eta[l], g.pg, g.neg, val[l], der[l]);
    for (int c = 0; c < D; ++c) x[c] = 0.0;
    for (int i = 0; i < D * D; ++i) J[i] = 0.0;
    const int m = g.neg + g.pg;  // basis functions per direction
    int idx[D];
    for (int l = 0; l < D; ++l) idx[l] = 0;
    while (true) {
        long long row = 0, stride = 1;
        for (int l = 0; l < D; ++l) {
            row += (first[l] + idx[l]) * stride;
            stride *= m;
        }
        double w = 1.0;
        for (int l = 0; l < D; ++l) w *= val[l][idx[l]];
        for (int r = 0; r < D; ++r) x[r] += w * g.cp[row + g.ncp * r];
        for (int c = 0; c < D; ++c) {
            double wc = 1.0;
            for (int l = 0; l < D; ++l) wc *= (l == c) ? der[l][idx[l]] : val[l][idx[l]];
            for (int r = 0; r < D; ++r) J[r + D * c] += wc * g.cp[row + g.ncp * r];
        }
        int l = 0;
        while (l < D && ++idx[l] > g.pg) idx[l++] = 0;
        if (l == D) break;
    }
}

template <int D>
__device__ __forceinline__ double det_inv(const double* J, double* Ji) {
    if (D == 1) {
        Ji[0] = 1.0 / J[0];
        return J[0];
    } else if (D == 2) {
        const double det = J[0] * J[3] - J[2] * J[1];
        Ji[0] = J[3] / det;
        Ji[3] = J[0] / det;
        Ji[2] = -J[2] / det;
        Ji[1] = -J[1] / det;
        return det;
    } else {
        auto a = [&](int r, int c) { return J[r + 3 * c]; };
        const double det = a(0, 0) * (a(1, 1) * a(2, 2) - a(2, 1) * a(1, 2)) -
                           a(0, 1) * (a(1, 0) * a(2, 2) - a(2, 0) * a(1, 2)) +
                           a(0, 2) * (a(1, 0) * a(2, 1) - a(2, 0) * a(1, 1));
        Ji[0 + 3 * 0] = (a(1, 1) * a(2, 2) - a(1, 2) * a(2, 1)) / det;
        Ji[0 + 3 * 1] = -(a(0, 1) * a(2, 2) - a(0, 2) * a(2, 1)) / det;
        Ji[0 + 3 * 2] = (a(0, 1) * a(1, 2) - a(0, 2) * a(1, 1)) / det;
        Ji[1 + 3 * 0] = -(a(1, 0) * a(2, 2) - a(1, 2) * a(2, 0)) / det;
        Ji[1 + 3 * 1] = (a(0, 0) * a(2, 2) - a(0, 2) * a(2, 0)) / det;
        Ji[1 + 3 * 2] = -(a(0, 0) * a(1, 2) - a(0, 2) * a(1, 0)) / det;
        Ji[2 + 3 * 0] = (a(1, 0) * a(2, 1) - a(1, 1) * a(2, 0)) / det;
        Ji[2 + 3 * 1] = -(a(0, 0) * a(2, 1) - a(0, 1) * a(2, 0)) / det;
        Ji[2 + 3 * 2] = (a(0, 0) * a(1, 1) - a(0, 1) * a(1, 0)) / det;
        return det;
    }
}

}  // namespace geomdev
}  // namespace gpu
}  // namespace stiga
