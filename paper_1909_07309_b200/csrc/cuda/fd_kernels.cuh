// Device side of the extended-FD apply: FP64 tensor-core (DMMA m8n8k4) mode products and the
// time-fused (U_t^T -> block-arrowhead solve -> U_t) kernel.
//
// Reference ops replaced:
//   mode_product / KronFactor::{contract,apply_left}  kronop.cpp:27-73
//   arrowhead_solve / apply_pair_inverse               fdsolve.cpp:11-65
//   ExtendedFDPreconditioner::apply (D^-1/2 scalings)  fdsolve.cpp:155-164
#pragma once

#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include <vector>

namespace stiga {
namespace gpu {

constexpr int kMaxDim = 4;  // spatial directions supported by the device path (reference: d = 1..3)

/// Per-spatial-index data of the block-arrowhead solve (ArrowheadLU, fdsolve.hpp:17-31).
/// R_j^-1 is recomputed on the fly from Lambda_s instead of being stored.
struct ArrowParams {
    int d = 0;
    int n[kMaxDim] = {0, 0, 0, 0};          // spatial mode sizes (colex, n[0] fastest)
    const double* lam[kMaxDim] = {};        // per-direction eigenvalues Lambda_l
    const double* S_inv = nullptr;          // N_s
    const double* pair_c = nullptr;         // gamma^2/nu * lambda_j^2  (fdsolve.cpp:118)
    const double* pair_c1 = nullptr;        // gamma/nu * lambda_j      (fdsolve.cpp:16)
    const double* pair_c1sq = nullptr;      // c1 * c1 / nu             (fdsolve.cpp:17, the reference's quirk)
    const double* pair_gg = nullptr;        // gamma * g[2j], gamma * g[2j+1] (2 per pair)
    const double* g = nullptr;              // n_t - 1 coupling entries
    int npairs = 0, zero_count = 0, n_t = 0;
    double gamma = 0.0, nu = 0.0, inv_nu = 0.0;
    long long s_off = 0;  // global index of local spatial index 0 (sharded apply)
    int debug = 0;  // bit 0: skip the arrowhead (Y = U_t U_t^T X); debugging aid
};

/// Geometry of one mode product over a colex tensor: fibers are indexed by
/// c = l + L*r (l < L, r < R); element j of fiber c sits at l + L*(j + n*r).
struct ModeGeom {
    long long L = 1;      // product of the sizes before the mode
    long long ncols = 0;  // L * R
    int n = 0;            // input mode size (contraction length)
    int m = 0;            // output mode size (rows of J; == n for the square FD factors)
};

/// Peer-memory scatter epilogue of the time-sharded apply: instead of storing to the
/// local output, the kernel stores every output element straight into the receive buffer of the
/// rank that owns it (NVLink P2P stores through pointers opened with CUDA IPC; local pointers for
/// virtual ranks), which fuses the all-to-all transpose into the producing product.
///   forward (by_time = 0, last spatial mode of a time slab): a = spatial index l + L*i, b = local
///     time slice r; owner q = the rank whose spatial range [off[q], off[q+1]) holds a;
///   backward (by_time = 1, time mode of a spatial slab): a = local spatial index l, b = time slice
///     i; owner q = the rank whose time range holds b.
/// Destination: ptr[q] + (a - (by_time ? 0 : off[q]) + a_shift) + ld[q] * (b - (by_time ? off[q] : 0) + b_shift).
constexpr int kMaxRanks = 8;
struct Scatter {
    int G = 0;        // ranks (1..kMaxRanks)
    int by_time = 0;  // owner coordinate: 0 = a (spatial), 1 = b (time)
    long long off[kMaxRanks + 1] = {};
    long long ld[kMaxRanks] = {};
    long long a_shift = 0, b_shift = 0;
    double* ptr[kMaxRanks] = {};
};

/// Kernel tiling chosen on the host (choose_mode_tiling / choose_time_tiling).
/// One CTA computes MI*WM*8 rows (a "row block") x BN fibers; warps are WM x WN, each owning
/// MI 8-row strips x NI 8-fiber tiles.  J is streamed in 16-column chunks through `nstage`
/// cp.async stages together with the matching 16-row chunk of the fiber tile.
struct Tiling {
    int MI = 1, WM = 1, NI = 2, WN = 4;
    int S = 1;        // 8-row strips covering m (ceil(m/8))
    int RB = 1;       // row blocks (mode kernel only; the time kernel keeps all rows in one CTA)
    int MpB = 8;      // J rows per CTA = 8*MI*WM
    int Mp = 8;       // padded rows of the uploaded J = RB*MpB
    int Kp = 4;       // padded contraction length = round_up(n, 4)
    int BN = 64;      // fibers per CTA = 8*NI*WN (power of two)
    int LDX = 68;     // smem row stride of a fiber chunk (== 4 mod 16 doubles)
    int Zrows = 0;    // time kernel: rows of the resident Z tile (= Kp)
    int nstage = 3;
    int fold = 0;     // 1: folded (centrosymmetric) product, fold_kernels.cu; 2: the resident-factor persistent
                      // folded kernel, fold_res.cu; MI/RB/Mp/Kp refer to the folded matrices
    int res = 0;      // 1: dense resident-factor persistent kernel (dense_res.cu); 2: resident time kernel
                      // (time_res.cu); MI = strips per warp,
                      // WM = strip groups, WN = fiber groups, MpB = rows per row block
    size_t smem = 0;
    int ctas_per_sm = 1;
    int threads() const { return 32 * WM * WN; }
};

Tiling choose_mode_tiling(int m, int n, bool prescale);  // m output rows, n contraction length
Tiling choose_time_tiling(int n_t);
/// All feasible tilings, best heuristic first (setup autotunes over the leading ones).
std::vector<Tiling> mode_tiling_candidates(int m, int n);
std::vector<Tiling> time_tiling_candidates(int n_t);

/// Y = (I (x) J (x) I) X along one mode.  J is row-major, zero padded to (t.Mp x t.Kp).
/// post_scale (optional) multiplies Y elementwise in the register epilogue (the D^-1/2 post-scale).
/// pre_scale (optional) multiplies X elementwise before the product (the D^-1/2 pre-scale, staged
/// beside each fiber chunk); needs prescale_fits(t).
/// sc (optional): scatter the output to the owners' receive buffers instead of Y (Y unused; no
/// pre/post scale).
cudaError_t launch_mode_product(const Tiling& t, const ModeGeom& g, const double* X, double* Y,
                                const double* Jpad, const double* post_scale, cudaStream_t stream,
                                const double* pre_scale = nullptr, const Scatter* sc = nullptr);
/// Dynamic smem of the pre-scaled mode kernel for tiling t, and whether it fits one CTA.
size_t prescale_smem(const Tiling& t);
bool prescale_fits(const Tiling& t);

/// Folded mode products of a centrosymmetric direction (fold_kernels.cu): half the FLOPs of the
/// dense product.  Jfold holds the two folded matrices, each row-major zero-padded t.Mp x t.Kp,
/// the second at offset t.Mp*t.Kp: forward (U^T) [A_e; A_o], backward (U) [A_p; A_q].
/// post_scale (backward only) multiplies the outputs elementwise.
/// pre_scale (forward only) multiplies both staged fiber chunks by D^-1/2 as the fold is formed.
std::vector<Tiling> fold_tiling_candidates(int n);
/// sc (forward, WM = 2 tilings only): scatter epilogue of the fused all-to-all (Scatter above).
cudaError_t launch_fold_product(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jfold,
                                bool forward, const double* post_scale, cudaStream_t stream,
                                const double* pre_scale = nullptr, const Scatter* sc = nullptr);
size_t fold_prescale_smem(const Tiling& t);
/// Dense resident-factor persistent mode product (dense_res.cu, Tiling::res == 1), candidates
/// for an m x n factor (the fused D^-1/2 pre-scale needs its own smem: prescale = true).
std::vector<Tiling> mode_res_candidates(int m, int n, bool prescale);
/// Resident-U_t persistent time kernel (time_res.cu, Tiling::res == 2): U_t^T -> arrowhead -> U_t
/// with one resident copy of U_t, two CTAs per SM; n_t up to ~110.
std::vector<Tiling> time_res_candidates(int n_t);
cudaError_t launch_time_res(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J_pad,
                            const ArrowParams& ap, cudaStream_t stream);
size_t mode_res_smem(const Tiling& t, bool prescale);
cudaError_t launch_mode_res(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                            const double* post, const double* pre, cudaStream_t st);
/// Resident-factor persistent folded product (fold_res.cu, Tiling::fold == 2): both folded matrices in
/// shared memory for the whole launch, one CTA per SM, warp-specialised cp.async/mbarrier pipeline.
/// Candidates for n with 4 <= ceil(ceil(n/2)/8) <= 11; no pre-scale / scatter epilogue.
std::vector<Tiling> fold_res_candidates(int n, int Mp_hint);
cudaError_t launch_fold_res(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jfold,
                            bool forward, const double* post_scale, cudaStream_t stream,
                            const double* pre_scale = nullptr);
size_t fold_res_prescale_smem(const Tiling& t);

/// Standalone block-arrowhead solve X = (gamma Delta_t (x) I + nu I (x) Lambda_s)^-1 Z on the
/// time-eigen-coordinate tensor (N_s x n_t, time slowest); used when the time direction runs as
/// three passes (U_t^T product, arrowhead, U_t product) instead of the fused kernel.
cudaError_t launch_arrowhead(const double* Z, double* X, long long Ns, const ArrowParams& ap, cudaStream_t stream);

/// Time-fused kernel: per spatial index, Z = U_t^T x, arrowhead solve, y = U_t Z.
/// Jt_pad = U_t^T padded, J_pad = U_t padded (both row-major Mp x Kp).
cudaError_t launch_time_fused(const Tiling& t, const ModeGeom& g, const double* X, double* Y,
                              const double* Jt_pad, const double* J_pad, const ArrowParams& ap,
                              cudaStream_t stream, const Scatter* sc = nullptr);

/// dst[r*dld + c] = src[r*sld + c] for r < rows, c < cols (pack/unpack of the sharded transposes).
cudaError_t launch_copy_blocks(const double* src, long long sld, double* dst, long long dld, long long rows,
                               long long cols, cudaStream_t stream);

/// Elementwise y = a .* x (the D^-1/2 post-scale of the last backward pass).
cudaError_t launch_scale(const double* a, const double* x, double* y, long long n, cudaStream_t stream);

}  // namespace gpu
}  // namespace stiga
