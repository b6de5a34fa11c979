// Space-time quadrature-grid kernels: the right-hand side b_ of SpaceTimeSystem (assemble_rhs,
// assembly.cpp:413-504) and the error norms of compute_errors (problems.cpp:305-402), both
// sum-factorized over the tensor Gauss grid instead of the reference's element loops:
//
//   b = (B_t^T (x) B_d^T (x) ... (x) B_1^T) F,   F(q_s, q_t) = w_s det J T w_t f(F(eta_s), T tau_t)
//   V = (B_t (x) B_d (x) ... (x) B_1) c           (and one derivative factor for grad / d/dt)
//
// with B_l the banded collocation matrices of the 1D spaces at the Gauss points (p+1 non-zeros per
// row, problems.cpp:35-49).  Time points are processed in batches so the grid tensors stay bounded.
#pragma once

#include <cuda_runtime.h>

#include "physical.cuh"

namespace stiga {
namespace gpu {

/// Manufactured source / exact-solution kinds of the problem catalog (problems.cpp:131-241).
enum SourceKind : int { kSrcNone = 0, kSrcIdentity = 1, kSrcAnnulus = 2, kSrcSeparableNu = 3 };

/// Spatial Gauss grid geometry, direction 0 fastest (Q_l points per direction): x (d planes of Nq),
/// wdet = (prod_l w_l) det J, JinvT (d*d planes, column-major J^-T).  Points with det J <= 0 set *bad.
/// g supplies the spline map (pg, neg, cp, ncp); JinvT may be null.
cudaError_t launch_qgrid_geometry(const PhysicalDesc& g, const double* const* qnode, const double* const* qweight,
                                  const int* Q, double* x, double* wdet, double* JinvT, int* bad, cudaStream_t st);

/// F[js + Nq*k] = (wdet[js] T) tweight[k] f(x_js, T tnode[k]) for k < nb (time nodes of the batch).
cudaError_t launch_rhs_eval(int d, int kind, long long Nq, const double* x, const double* wdet, const double* tnode,
                            const double* tweight, int nb, double T, double* F, cudaStream_t st);

/// Banded collocation product along the middle mode of an (L, ., R) tensor.
///  forward  : out(L, nout, R)[l, q, r] = sum_a tab[(qoff+q) p1 + a] in[l, first[qoff+q] + a, r]  (in: nin rows)
///  transpose: out(L, nout, R)[l, i, r] = beta out + sum_{qg in [tlo[i], thi[i]) & [qoff, qoff+nin)}
///             tab[qg p1 + i - first[qg]] in[l, qg - qoff, r]                                     (in: nin = batch rows)
cudaError_t launch_colloc(long long L, int nin, long long R, int nout, const int* first, const double* tab, int p1,
                          const int* tlo, const int* thi, int qoff, bool transpose, double beta, const double* in,
                          double* out, cudaStream_t st);

/// Per-block partial sums (4 per block: l2 num, l2 den, X num, X den) of compute_errors over a batch
/// of nb time points: V, G[l], Vt are (Nq, nb) grids of u_h, its parametric gradient and d/dtau.
cudaError_t launch_error_terms(int d, int kind, long long Nq, int nb, const double* x, const double* wdet,
                               const double* JinvT, const double* V, const double* G0, const double* G1,
                               const double* G2, const double* Vt, const double* tnode, const double* tweight,
                               double T, double wt_dt, double nu, double* partial, int nblocks, cudaStream_t st);

}  // namespace gpu
}  // namespace stiga
