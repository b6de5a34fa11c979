// cuSOLVER symmetric eigensolver (host/eig_device.cpp): the sym_eig backend of the device setup.
#pragma once

#include "linalg.hpp"

namespace stiga {

/// cusolverDnDsyevd on the calling thread's current CUDA device; ascending w, orthonormal Q.
void sym_eig_cusolver(const DenseMatrix& A, Vector& w, DenseMatrix& Q);

}  // namespace stiga
