// Geometry map, problem catalog and A^G coefficient pieces (see geometry.hpp for the reference map).
#include "geometry.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>
#include <thread>

namespace stiga {

namespace {

constexpr double kPi = 3.14159265358979323846;

bool advance(std::vector<int>& idx, const std::vector<int>& dims) {
    for (size_t l = 0; l < idx.size(); ++l) {
        if (++idx[l] < dims[l]) return true;
        idx[l] = 0;
    }
    return false;
}

double det_small(const double* J, int d) {  // column-major d x d
    if (d == 1) return J[0];
    if (d == 2) return J[0] * J[3] - J[2] * J[1];
    return J[0] * (J[4] * J[8] - J[7] * J[5]) - J[3] * (J[1] * J[8] - J[7] * J[2]) + J[6] * (J[1] * J[5] - J[4] * J[2]);
}

void inv_small(const double* J, int d, double det, double* Ji) {  // column-major inverse
    if (d == 1) {
        Ji[0] = 1.0 / J[0];
        return;
    }
    if (d == 2) {
        Ji[0] = J[3] / det;
        Ji[3] = J[0] / det;
        Ji[2] = -J[2] / det;
        Ji[1] = -J[1] / det;
        return;
    }
    auto a = [&](int r, int c) { return J[r + 3 * c]; };
    double C[9];
    C[0 + 3 * 0] = a(1, 1) * a(2, 2) - a(1, 2) * a(2, 1);
    C[0 + 3 * 1] = -(a(0, 1) * a(2, 2) - a(0, 2) * a(2, 1));
    C[0 + 3 * 2] = a(0, 1) * a(1, 2) - a(0, 2) * a(1, 1);
    C[1 + 3 * 0] = -(a(1, 0) * a(2, 2) - a(1, 2) * a(2, 0));
    C[1 + 3 * 1] = a(0, 0) * a(2, 2) - a(0, 2) * a(2, 0);
    C[1 + 3 * 2] = -(a(0, 0) * a(1, 2) - a(0, 2) * a(1, 0));
    C[2 + 3 * 0] = a(1, 0) * a(2, 1) - a(1, 1) * a(2, 0);
    C[2 + 3 * 1] = -(a(0, 0) * a(2, 1) - a(0, 1) * a(2, 0));
    C[2 + 3 * 2] = a(0, 0) * a(1, 1) - a(0, 1) * a(1, 0);
    for (int i = 0; i < 9; ++i) Ji[i] = C[i] / det;
}

// Colex mode product on the host: y = (I (x) A (x) I) x along `mode`, A rows x cols (column-major).
std::vector<double> host_mode_product(const std::vector<double>& x, std::vector<Index>& dims, const DenseMatrix& A,
                                      int mode) {
    Index left = 1, right = 1;
    for (int l = 0; l < mode; ++l) left *= dims[l];
    for (size_t l = mode + 1; l < dims.size(); ++l) right *= dims[l];
    const Index n = dims[mode], m = A.rows;
    std::vector<double> y(static_cast<size_t>(left * m * right), 0.0);
    for (Index r = 0; r < right; ++r)
        for (Index j = 0; j < n; ++j)
            for (Index i = 0; i < m; ++i) {
                const double a = A(i, j);
                if (a == 0.0) continue;
                const double* xs = x.data() + left * (j + n * r);
                double* ys = y.data() + left * (i + m * r);
                for (Index l = 0; l < left; ++l) ys[l] += a * xs[l];
            }
    dims[mode] = m;
    return y;
}

DenseMatrix collocation_full(const KnotVector& kv, const std::vector<double>& pts) {
    const int m = kv.num_basis(), p = kv.degree();
    DenseMatrix B(static_cast<Index>(pts.size()), m);
    std::vector<double> buf(p + 1);
    for (size_t q = 0; q < pts.size(); ++q) {
        const int first = kv.eval_basis(pts[q], 0, buf.data());
        for (int r = 0; r <= p; ++r) B(static_cast<Index>(q), first + r) = buf[r];
    }
    return B;
}

std::vector<double> linspace01(int n) {
    std::vector<double> x(n);
    for (int i = 0; i < n; ++i) x[i] = static_cast<double>(i) / (n - 1);
    return x;
}

void check_positive(double det, const double* eta, int d, const char* what) {
    if (det > 0.0) return;
    std::string msg = std::string(what) + ": det J_F = " + std::to_string(det) + " <= 0 at eta = (";
    for (int l = 0; l < d; ++l) msg += (l ? ", " : "") + std::to_string(eta[l]);
    throw std::runtime_error(msg + ")");
}

}  // namespace

GeometryMap::GeometryMap(std::vector<KnotVector> kvs, DenseMatrix cp) : kvs_(std::move(kvs)), cp_(std::move(cp)) {
    if (kvs_.empty() || kvs_.size() > 3)
        throw std::invalid_argument("GeometryMap: spatial dimension must be 1, 2 or 3");
    Index total = 1;
    strides_.resize(kvs_.size());
    for (size_t l = 0; l < kvs_.size(); ++l) {
        strides_[l] = total;
        total *= kvs_[l].num_basis();
    }
    if (cp_.rows != total || cp_.cols != static_cast<Index>(kvs_.size()))
        throw std::invalid_argument("GeometryMap: control point array has wrong shape");
}

GeometryMap GeometryMap::identity(int d) {
    std::vector<KnotVector> kvs(d, KnotVector::uniform_open(1, 1));
    const Index total = Index(1) << d;
    DenseMatrix cp(total, d);
    for (Index i = 0; i < total; ++i)
        for (int l = 0; l < d; ++l) cp(i, l) = static_cast<double>((i >> l) & 1);
    return GeometryMap(std::move(kvs), std::move(cp));
}

void GeometryMap::value(const double* eta, double* x) const {
    const int d = dim();
    int first[3];
    double val[3][16];
    for (int l = 0; l < d; ++l) first[l] = kvs_[l].eval_basis(eta[l], 0, val[l]);
    for (int c = 0; c < d; ++c) x[c] = 0.0;
    int idx[3] = {0, 0, 0};
    while (true) {
        double w = 1.0;
        Index row = 0;
        for (int l = 0; l < d; ++l) {
            w *= val[l][idx[l]];
            row += (first[l] + idx[l]) * strides_[l];
        }
        for (int c = 0; c < d; ++c) x[c] += w * cp_(row, c);
        int l = 0;
        while (l < d && ++idx[l] > kvs_[l].degree()) idx[l++] = 0;
        if (l == d) break;
    }
}

void GeometryMap::jacobian(const double* eta, double* J) const {
    const int d = dim();
    int first[3];
    double val[3][16], der[3][16];
    for (int l = 0; l < d; ++l) {
        first[l] = kvs_[l].eval_basis(eta[l], 0, val[l]);
        kvs_[l].eval_basis(eta[l], 1, der[l]);
    }
    for (int i = 0; i < d * d; ++i) J[i] = 0.0;
    int idx[3] = {0, 0, 0};
    while (true) {
        Index row = 0;
        for (int l = 0; l < d; ++l) row += (first[l] + idx[l]) * strides_[l];
        for (int c = 0; c < d; ++c) {
            double w = 1.0;
            for (int l = 0; l < d; ++l) w *= (l == c) ? der[l][idx[l]] : val[l][idx[l]];
            for (int r = 0; r < d; ++r) J[r + d * c] += w * cp_(row, r);
        }
        int l = 0;
        while (l < d && ++idx[l] > kvs_[l].degree()) idx[l++] = 0;
        if (l == d) break;
    }
}

GeometryMap fit_geometry(const MapFn& map, int d, int p_g, int n_el, double* max_residual) {
    if (d < 1 || d > 3) throw std::invalid_argument("fit_geometry: d must be 1, 2 or 3");
    std::vector<KnotVector> kvs;
    std::vector<int> nsamp(d);
    std::vector<DenseMatrix> colloc, projector;
    for (int l = 0; l < d; ++l) {
        kvs.push_back(KnotVector::uniform_open(p_g, n_el));
        const int m = kvs[l].num_basis();
        nsamp[l] = std::max(4 * m, 32);
        DenseMatrix B = collocation_full(kvs[l], linspace01(nsamp[l]));
        DenseMatrix BtB = matmul_tn(B, B), L;
        if (!cholesky(BtB, L)) throw std::runtime_error("fit_geometry: singular collocation normal matrix");
        DenseMatrix P = B.transpose();  // (B^T B)^-1 B^T via the Cholesky factor
        trsm_lower(L, P);
        trsm_lower_t(L, P);
        colloc.push_back(std::move(B));
        projector.push_back(std::move(P));
    }
    Index n_pts = 1;
    for (int l = 0; l < d; ++l) n_pts *= nsamp[l];
    std::vector<std::vector<double>> samples(d, std::vector<double>(static_cast<size_t>(n_pts)));
    {
        std::vector<int> idx(d, 0);
        Index flat = 0;
        double eta[3], x[3];
        do {
            for (int l = 0; l < d; ++l) eta[l] = static_cast<double>(idx[l]) / (nsamp[l] - 1);
            map(eta, x);
            for (int c = 0; c < d; ++c) samples[c][flat] = x[c];
            ++flat;
        } while (advance(idx, nsamp));
    }
    Index m_total = 1;
    for (int l = 0; l < d; ++l) m_total *= kvs[l].num_basis();
    DenseMatrix cp(m_total, d);
    double maxres = 0.0;
    std::vector<double> res2(static_cast<size_t>(n_pts), 0.0);
    for (int c = 0; c < d; ++c) {
        std::vector<Index> dims(nsamp.begin(), nsamp.end());
        std::vector<double> t = samples[c];
        for (int l = 0; l < d; ++l) t = host_mode_product(t, dims, projector[l], l);
        for (Index i = 0; i < m_total; ++i) cp(i, c) = t[i];
        for (int l = 0; l < d; ++l) t = host_mode_product(t, dims, colloc[l], l);
        for (Index i = 0; i < n_pts; ++i) res2[i] += (t[i] - samples[c][i]) * (t[i] - samples[c][i]);
    }
    for (double r : res2) maxres = std::max(maxres, std::sqrt(r));
    if (max_residual) *max_residual = maxres;
    GeometryMap F(std::move(kvs), std::move(cp));
    // reject maps whose fitted Jacobian loses positivity (problems.cpp:107-122)
    std::vector<QuadratureRule> rules;
    std::vector<int> npts(d);
    for (int l = 0; l < d; ++l) {
        rules.push_back(gauss_rule(F.knot_vectors()[l], p_g + 1));
        npts[l] = rules[l].num_points();
    }
    std::vector<int> idx(d, 0);
    double eta[3], J[9];
    do {
        for (int l = 0; l < d; ++l) eta[l] = rules[l].nodes[idx[l]];
        F.jacobian(eta, J);
        if (det_small(J, d) <= 0.0) throw std::runtime_error("fit_geometry: fitted Jacobian not positive on [0,1]^d");
    } while (advance(idx, npts));
    return F;
}

ProblemSpec make_problem(const std::string& id) {
    ProblemSpec prob;
    prob.name = id;
    if (id == "identity-interval-1d" || id == "identity-square-2d" || id == "identity-cube-3d") {
        prob.d = id == "identity-interval-1d" ? 1 : (id == "identity-square-2d" ? 2 : 3);
        prob.geometry = GeometryMap::identity(prob.d);
    } else if (id == "quarter-annulus-2d") {  // problems.cpp:194-216
        prob.d = 2;
        prob.geometry = fit_geometry(
            [](const double* eta, double* x) {
                const double r = 1.0 + eta[0], th = 0.5 * kPi * eta[1];
                x[0] = r * std::cos(th);
                x[1] = r * std::sin(th);
            },
            2, 3, 8);
    } else if (id == "separable-nu-2d") {  // problems.cpp:220-240
        prob.d = 2;
        prob.geometry = GeometryMap::identity(2);
        prob.nu_s = [](const double* x) { return 50.5 + 49.5 * x[1] / std::hypot(x[0], x[1]); };
        prob.nu_t = [](double t) { return 1.0 + 50.0 * (1.0 + std::cos(t / (2.0 * kPi))); };
    } else if (id == "deformed-cube-3d") {  // BASELINE.json configs[3]
        prob.d = 3;
        prob.geometry = fit_geometry(
            [](const double* eta, double* x) {
                const double b = 0.1 * std::sin(kPi * eta[0]) * std::sin(kPi * eta[1]) * std::sin(kPi * eta[2]);
                for (int l = 0; l < 3; ++l) x[l] = eta[l] + b;
            },
            3, 3, 8);
        prob.nu_s = [](const double* x) { return 1.0 + 0.5 * std::sin(2.0 * kPi * x[0]) * std::cos(2.0 * kPi * x[1]); };
        prob.gamma_s = [](const double* x) { return 1.0 + 0.25 * x[2]; };
    } else {
        throw std::invalid_argument("make_problem: unknown problem id '" + id + "'");
    }
    return prob;
}

std::vector<double> coefficient_diagonal_samples(const std::vector<KnotVector>& kvs, const GeometryMap& F,
                                                 const FieldFn& nu_s, const FieldFn& gamma_s) {
    const int d = static_cast<int>(kvs.size());
    if (F.dim() != d) throw std::invalid_argument("coefficient_diagonal_samples: geometry dimension mismatch");
    std::vector<int> nel(d);
    Index n_elems = 1;
    for (int l = 0; l < d; ++l) {
        nel[l] = kvs[l].num_elements();
        n_elems *= nel[l];
    }
    std::vector<double> out(static_cast<size_t>(n_elems * (d + 1)));
    std::vector<int> e(d, 0);
    Index flat = 0;
    double eta[3], J[9], Ji[9], x[3];
    do {
        for (int l = 0; l < d; ++l) {
            const auto ab = kvs[l].element(e[l]);
            eta[l] = 0.5 * (ab.first + ab.second);
        }
        F.jacobian(eta, J);
        const double det = det_small(J, d);
        check_positive(det, eta, d, "geometry error");
        inv_small(J, d, det, Ji);
        double nu = 1.0, gam = 1.0;
        if (nu_s || gamma_s) {
            F.value(eta, x);
            if (nu_s) nu = nu_s(x);
            if (gamma_s) gam = gamma_s(x);
        }
        for (int l = 0; l < d; ++l) {
            double cll = 0.0;  // (J^-1 J^-T)_{ll} = sum_k (J^-1)_{lk}^2
            for (int k = 0; k < d; ++k) cll += Ji[l + d * k] * Ji[l + d * k];
            out[flat + l * n_elems] = cll * det * nu;
        }
        out[flat + d * n_elems] = det * gam;
        ++flat;
    } while (advance(e, nel));
    return out;
}

SeparableCoefficients separate_variables(const std::vector<double>& samples, const std::vector<int>& nel) {
    const int d = static_cast<int>(nel.size());
    Index n_elems = 1;
    for (int l = 0; l < d; ++l) n_elems *= nel[l];
    if (d < 1 || static_cast<Index>(samples.size()) != n_elems * (d + 1))
        throw std::invalid_argument("separate_variables: samples must have dims (n_el_1..n_el_d, d+1)");
    for (double v : samples)
        if (!(v > 0.0)) throw std::invalid_argument("separate_variables: all samples must be positive");
    auto slice = [&](int s) { return samples.data() + s * n_elems; };
    SeparableCoefficients out;
    out.phi.assign(d, {});
    out.Phi.assign(d, {});
    for (int l = 0; l < d; ++l) {
        out.phi[l].assign(nel[l], 1.0);
        out.Phi[l].assign(nel[l], 1.0);
    }
    const double* G = slice(d);
    out.converged = false;
    for (int sweep = 0; sweep < 50; ++sweep) {
        double max_rel = 0.0;
        for (int l = 0; l < d; ++l) {
            std::vector<double> num(nel[l], 0.0), den(nel[l], 0.0);
            std::vector<int> m(d, 0);
            Index flat = 0;
            do {
                double w = 1.0;
                for (int k = 0; k < d; ++k)
                    if (k != l) w *= out.phi[k][m[k]];
                num[m[l]] += G[flat] * w;
                den[m[l]] += w * w;
                ++flat;
            } while (advance(m, nel));
            for (int i = 0; i < nel[l]; ++i) {
                const double next = num[i] / den[i];
                max_rel = std::max(max_rel, std::abs(next - out.phi[l][i]) / std::abs(out.phi[l][i]));
                out.phi[l][i] = next;
            }
        }
        out.sweeps = sweep + 1;
        if (max_rel <= 1e-10) {
            out.converged = true;
            break;
        }
    }
    for (int l = 1; l < d; ++l) {  // gauge: unit geometric mean except the first factor
        double logsum = 0.0;
        for (double v : out.phi[l]) logsum += std::log(v);
        const double g = std::exp(logsum / nel[l]);
        for (double& v : out.phi[l]) v /= g;
        for (double& v : out.phi[0]) v *= g;
    }
    for (int l = 0; l < d; ++l) {
        std::vector<double> acc(nel[l], 0.0);
        std::vector<int> cnt(nel[l], 0);
        const double* E = slice(l);
        std::vector<int> m(d, 0);
        Index flat = 0;
        do {
            double w = 1.0;
            for (int k = 0; k < d; ++k)
                if (k != l) w *= out.phi[k][m[k]];
            acc[m[l]] += E[flat] / w;
            cnt[m[l]] += 1;
            ++flat;
        } while (advance(m, nel));
        for (int i = 0; i < nel[l]; ++i) out.Phi[l][i] = acc[i] / cnt[i];
    }
    out.residuals.assign(d + 1, 0.0);
    for (int s = 0; s <= d; ++s) {
        const double* E = slice(s);
        double num = 0.0, den = 0.0;
        std::vector<int> m(d, 0);
        Index flat = 0;
        do {
            double fit = 1.0;
            for (int k = 0; k < d; ++k) fit *= (k == s) ? out.Phi[k][m[k]] : out.phi[k][m[k]];
            num += (E[flat] - fit) * (E[flat] - fit);
            den += E[flat] * E[flat];
            ++flat;
        } while (advance(m, nel));
        out.residuals[s] = std::sqrt(num / den);
    }
    return out;
}

void physical_diagonals(const std::vector<SplineSpace1D>& spaces, const GeometryMap& F, int q, const FieldFn& nu_s,
                        const FieldFn& gamma_s, std::vector<double>& dK, std::vector<double>& dM) {
    const int d = static_cast<int>(spaces.size());
    if (F.dim() != d) throw std::invalid_argument("assemble_spatial_physical: geometry dimension mismatch");
    std::vector<QuadratureRule> quads;
    std::vector<int> n(d), nel(d), loc(d);
    std::vector<std::vector<double>> val(d), der(d);  // per 1D quad point: p+1 values / derivatives
    std::vector<std::vector<int>> first(d);
    Index n_total = 1;
    for (int l = 0; l < d; ++l) {
        quads.push_back(gauss_rule(spaces[l].knot_vector(), q));
        n[l] = spaces[l].dim();
        nel[l] = quads[l].num_elements;
        loc[l] = spaces[l].degree() + 1;
        n_total *= n[l];
        const int np = quads[l].num_points();
        val[l].resize(static_cast<size_t>(np) * loc[l]);
        der[l].resize(static_cast<size_t>(np) * loc[l]);
        first[l].resize(np);
        for (int qp = 0; qp < np; ++qp) {
            first[l][qp] = spaces[l].eval_active(quads[l].nodes[qp], 0, &val[l][qp * loc[l]]);
            spaces[l].eval_active(quads[l].nodes[qp], 1, &der[l][qp * loc[l]]);
        }
    }
    std::vector<Index> stride(d, 1);
    for (int l = 1; l < d; ++l) stride[l] = stride[l - 1] * n[l - 1];
    const int nthreads = std::max(1, std::min<int>(static_cast<int>(std::thread::hardware_concurrency()), nel[d - 1]));
    std::vector<std::vector<double>> pK(nthreads, std::vector<double>(static_cast<size_t>(n_total), 0.0));
    std::vector<std::vector<double>> pM(nthreads, std::vector<double>(static_cast<size_t>(n_total), 0.0));
    std::vector<std::string> errors(nthreads);
    auto work = [&](int tid) {
        try {
            std::vector<int> enel(nel);
            enel[d - 1] = 1;
            std::vector<int> dimsq(d, q), dimsa(loc);
            double eta[3], J[9], Ji[9], x[3];
            for (int elast = tid; elast < nel[d - 1]; elast += nthreads) {
                std::vector<int> e(d, 0);
                do {
                    e[d - 1] = elast;
                    std::vector<int> jq(d, 0);
                    do {
                        double w = 1.0;
                        int qp[3];
                        for (int l = 0; l < d; ++l) {
                            qp[l] = e[l] * q + jq[l];
                            eta[l] = quads[l].nodes[qp[l]];
                            w *= quads[l].weights[qp[l]];
                        }
                        F.jacobian(eta, J);
                        const double det = det_small(J, d);
                        check_positive(det, eta, d, "geometry error");
                        inv_small(J, d, det, Ji);
                        double nu = 1.0, gam = 1.0;
                        if (nu_s || gamma_s) {
                            F.value(eta, x);
                            if (nu_s) nu = nu_s(x);
                            if (gamma_s) gam = gamma_s(x);
                        }
                        const double wk = w * det * nu, wm = w * det * gam;
                        std::vector<int> a(d, 0);
                        do {
                            Index g = 0;
                            bool ok = true;
                            double v = 1.0, gp[3];
                            for (int l = 0; l < d; ++l) {
                                const int act = first[l][qp[l]] + a[l];
                                if (act < 0 || act >= n[l]) {
                                    ok = false;
                                    break;
                                }
                                g += act * stride[l];
                                v *= val[l][qp[l] * loc[l] + a[l]];
                            }
                            if (!ok) continue;
                            for (int c = 0; c < d; ++c) {
                                double t = 1.0;
                                for (int l = 0; l < d; ++l)
                                    t *= (l == c) ? der[l][qp[l] * loc[l] + a[l]] : val[l][qp[l] * loc[l] + a[l]];
                                gp[c] = t;
                            }
                            double gg = 0.0;  // |J^-T grad_param|^2
                            for (int r = 0; r < d; ++r) {
                                double s = 0.0;
                                for (int c = 0; c < d; ++c) s += Ji[c + d * r] * gp[c];
                                gg += s * s;
                            }
                            pK[tid][g] += wk * gg;
                            pM[tid][g] += wm * v * v;
                        } while (advance(a, dimsa));
                    } while (advance(jq, dimsq));
                } while (advance(e, enel));
            }
        } catch (const std::exception& ex) {
            errors[tid] = ex.what();
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < nthreads; ++t) pool.emplace_back(work, t);
    for (auto& th : pool) th.join();
    for (const auto& err : errors)
        if (!err.empty()) throw std::runtime_error(err);
    dK.assign(static_cast<size_t>(n_total), 0.0);
    dM.assign(static_cast<size_t>(n_total), 0.0);
    for (int t = 0; t < nthreads; ++t)
        for (Index i = 0; i < n_total; ++i) {
            dK[i] += pK[t][i];
            dM[i] += pM[t][i];
        }
}

void time_matrices(const ProblemSpec& prob, int p, int n_el, DenseMatrix& Wt, DenseMatrix& Mt) {
    const double T = prob.T;
    auto [W, Mplain] = assemble_time_matrices(p, n_el, T);
    Wt = std::move(W.m);
    const SplineSpace1D tspace = SplineSpace1D::temporal(p, n_el);
    const QuadratureRule tquad = gauss_rule(tspace.knot_vector(), p + 1);
    if (prob.nu_t || prob.gamma_t) {  // M_t carries nu_t/gamma_t (solver.cpp:119-125)
        const auto tw = [&](double tau) {
            const double nt = prob.nu_t ? prob.nu_t(T * tau) : 1.0;
            const double gt = prob.gamma_t ? prob.gamma_t(T * tau) : 1.0;
            return nt / gt;
        };
        BandedMatrix Mh = assemble_univariate_fn(tspace, tquad, 0, 0, tw);
        for (double& v : Mh.m.a) v *= T;
        Mt = std::move(Mh.m);
    } else {
        Mt = std::move(Mplain.m);
    }
}

void problem_field_kinds(const ProblemSpec& prob, int& nu_kind, int& gamma_kind) {
    nu_kind = gamma_kind = 0;  // gpu::kFieldOne
    if (prob.name == "separable-nu-2d") nu_kind = 1;
    if (prob.name == "deformed-cube-3d") {
        nu_kind = 2;
        gamma_kind = 3;
    }
}

int problem_source_kind(const ProblemSpec& prob) {
    if (prob.name.rfind("identity-", 0) == 0) return 1;
    if (prob.name == "quarter-annulus-2d") return 2;
    if (prob.name == "separable-nu-2d") return 3;
    return 0;  // deformed-cube-3d: BASELINE config 4 runs on a seeded RHS
}

void system_means(const ProblemSpec& prob, int p, int n_el, double& gamma_mean, double& nu_mean) {
    const int d = prob.d, q = p + 1;
    const double T = prob.T;
    std::vector<QuadratureRule> rules;
    std::vector<int> npts(d);
    for (int l = 0; l < d; ++l) {
        rules.push_back(gauss_rule(SplineSpace1D::spatial(p, n_el).knot_vector(), q));
        npts[l] = rules[l].num_points();
    }
    double vol = 0.0, g_int = 0.0, n_int = 0.0;
    std::vector<int> idx(d, 0);
    double eta[3], x[3], J[9];
    do {
        double w = 1.0;
        for (int l = 0; l < d; ++l) {
            eta[l] = rules[l].nodes[idx[l]];
            w *= rules[l].weights[idx[l]];
        }
        prob.geometry.jacobian(eta, J);
        const double det = det_small(J, d);
        prob.geometry.value(eta, x);
        vol += w * det;
        g_int += w * det * (prob.gamma_s ? prob.gamma_s(x) : 1.0);
        n_int += w * det * (prob.nu_s ? prob.nu_s(x) : 1.0);
    } while (advance(idx, npts));
    const QuadratureRule tquad = gauss_rule(SplineSpace1D::temporal(p, n_el).knot_vector(), q);
    double t_mean = 0.0;
    for (int qt = 0; qt < tquad.num_points(); ++qt) {
        const double tau = tquad.nodes[qt];
        const double nt = prob.nu_t ? prob.nu_t(T * tau) : 1.0;
        const double gt = prob.gamma_t ? prob.gamma_t(T * tau) : 1.0;
        t_mean += tquad.weights[qt] * (nt / gt);
    }
    gamma_mean = g_int / vol;
    nu_mean = n_int / vol * t_mean;
}

GeometryPreconditionerPieces geometry_preconditioner_pieces(const ProblemSpec& prob, int p, int n_el, bool want_D) {
    const int d = prob.d, q = p + 1;
    const double T = prob.T;
    GeometryPreconditionerPieces out;
    std::vector<SplineSpace1D> spaces;
    std::vector<KnotVector> kvs;
    for (int l = 0; l < d; ++l) {
        spaces.push_back(SplineSpace1D::spatial(p, n_el));
        kvs.push_back(spaces.back().knot_vector());
    }
    (void)T;
    time_matrices(prob, p, n_el, out.Wt, out.Mt);
    // separated coefficients and the weighted 1D factors (solver.cpp:114-119, 130-136)
    std::vector<int> nel(d, n_el);
    out.sep = separate_variables(coefficient_diagonal_samples(kvs, prob.geometry, prob.nu_s, prob.gamma_s), nel);
    for (int l = 0; l < d; ++l) {
        const QuadratureRule quad = gauss_rule(kvs[l], q);
        out.Kt.push_back(assemble_univariate(spaces[l], quad, 1, 1, &out.sep.Phi[l]).m);
        out.Mt_s.push_back(assemble_univariate(spaces[l], quad, 0, 0, &out.sep.phi[l]).m);
    }
    if (want_D) {  // D = diag(A) / diag(A~)  (solver.cpp:138-142)
        std::vector<double> dK, dM;
        physical_diagonals(spaces, prob.geometry, q, prob.nu_s, prob.gamma_s, dK, dM);
        const Index ns = static_cast<Index>(dK.size()), nt = out.Wt.rows;
        // A~ = kron_sum_terms(K~, M~, W_t, M_t, 1, 1): diag = prod diag(M~_l) diag(W_t) + sum_l ...
        std::vector<double> dMt(ns, 1.0);
        std::vector<std::vector<double>> dKl(d);
        {
            std::vector<double> acc(1, 1.0);
            for (int l = 0; l < d; ++l) {
                std::vector<double> next(acc.size() * out.Mt_s[l].rows);
                for (Index j = 0; j < out.Mt_s[l].rows; ++j)
                    for (size_t i = 0; i < acc.size(); ++i) next[j * acc.size() + i] = out.Mt_s[l](j, j) * acc[i];
                acc.swap(next);
            }
            dMt = acc;
        }
        std::vector<double> dSt(ns, 0.0);  // diag of sum_l (M~ .. K~_l .. M~)
        for (int l = 0; l < d; ++l) {
            std::vector<double> acc(1, 1.0);
            for (int k = 0; k < d; ++k) {
                const DenseMatrix& F = (k == l) ? out.Kt[k] : out.Mt_s[k];
                std::vector<double> next(acc.size() * F.rows);
                for (Index j = 0; j < F.rows; ++j)
                    for (size_t i = 0; i < acc.size(); ++i) next[j * acc.size() + i] = F(j, j) * acc[i];
                acc.swap(next);
            }
            for (Index i = 0; i < ns; ++i) dSt[i] += acc[i];
        }
        out.D.resize(static_cast<size_t>(ns * nt));
        for (Index t = 0; t < nt; ++t) {
            const double w = out.Wt(t, t), m = out.Mt(t, t);
            for (Index i = 0; i < ns; ++i) {
                const double num = 1.0 * (dM[i] * w) + 1.0 * (dK[i] * m);
                const double den = 1.0 * (dMt[i] * w) + 1.0 * (dSt[i] * m);
                out.D[t * ns + i] = num / den;
            }
        }
    }
    return out;
}

}  // namespace stiga
