// FP64 tensor-core kernels of the extended-FD apply (sm_100a).
//
// Every mode product is a batch of small GEMMs  Y_fiber = J * X_fiber  with J the n x n
// eigenvector factor (n = 16..260).  A CTA owns a row block of J (MI*WM 8-row strips) and
// BN = 16*WN fibers.  Both operands stream through a 2-3 stage cp.async pipeline in 16-wide
// contraction chunks (J chunk: rows x 16 from L2, fiber chunk: 16 x BN from HBM), the products
// run on the FP64 tensor cores (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4; 36.9 TF/s measured on
// B200 vs 34.0 TF/s for DFMA, profiles/r01_fp64_peak.txt) with fragments double-buffered in
// registers, and the accumulators are stored straight from registers (no smem epilogue), so
// several CTAs per SM overlap one tile's epilogue with another's main loop.  All per-chunk
// producer work is compile-time unrolled (element counts follow from MI/WM/WN) so the issue
// slots go to LDS + DMMA.
//
// The time-fused kernel keeps the whole n_t x BN tile of one CTA: Z = U_t^T X lands in shared
// memory, the block-arrowhead solve of fdsolve.cpp:24-65 (forward pair eliminations, diagonal
// Schur, back substitution) runs in place, and Z is the resident B operand of y = U_t Z; the
// time direction costs one HBM round trip instead of three.
#include "fd_mode_impl.cuh"

#include <cstdlib>
#include <string>

namespace stiga {
namespace gpu {

namespace {

cudaError_t dispatch_mode(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                          const double* post, const double* pre, cudaStream_t st, int* occ,
                          const Scatter* sc = nullptr) {
    if (sc) return dispatch_mode_scatter(t, g, X, J, st, occ, sc);
    if (pre) return dispatch_mode_v<true, false>(t, g, X, Y, J, post, pre, st, occ, nullptr);
    return dispatch_mode_v<false, false>(t, g, X, Y, J, post, nullptr, st, occ, nullptr);
}

}  // namespace

std::vector<Tiling> mode_tiling_candidates(int m, int n) {
    std::vector<std::pair<double, Tiling>> c;
    const int S = (m + 7) / 8;
    const int Kp = (n + 3) / 4 * 4;
    const int rb0 = (S + 12) / 13;
    for (int RB = rb0; RB <= std::min(S, rb0 + 3); ++RB) {
        const int MI = (S + RB - 1) / RB;
        if (MI > 13 || MI < 1) continue;
        if (RB > rb0 && (S + rb0 - 1) / rb0 == MI) continue;  // same MI as a smaller RB
        for (int WN : {4, 2})
        for (int ns : {3, 2}) {  // 2 stages: half the staging smem (the fused pre-scale doubles it)
            Tiling t;
            t.MI = MI;
            t.WM = 1;
            t.NI = 2;
            t.WN = WN;
            t.S = S;
            t.RB = RB;
            t.MpB = 8 * MI;
            t.Mp = RB * t.MpB;
            t.Kp = Kp;
            t.BN = 16 * WN;
            t.LDX = t.BN + 4;
            t.nstage = ns;
            t.smem = sizeof(double) * static_cast<size_t>(t.nstage) * (kBK * t.LDX + t.MpB * kLDJ);
            if (t.smem > kSmemPerCTA) continue;
            int occ = 0;
            dispatch_mode(t, ModeGeom{}, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &occ);
            t.ctas_per_sm = occ;
            if (occ < 1) continue;
            // strips past S are skipped, so padding costs only imbalance; each extra row block
            // re-stages the fiber tile
            const double eff = 0.85 + 0.15 * static_cast<double>(S) / (RB * MI);
            c.emplace_back(std::min(occ * t.WN, 16) * eff + 0.02 * WN - 0.05 * RB - (ns == 2 ? 0.3 : 0.0), t);
        }
    }
    // two warp rows per CTA (WM = 2): twice the rows of one fiber tile per CTA at the same registers
    // per thread -- fewer row blocks re-staging the fiber tile
    const int rb2 = (S + 15) / 16;
    for (int RB = rb2; RB <= std::min(S, rb2 + 2); ++RB) {
        const int MI = (S + 2 * RB - 1) / (2 * RB);
        if (MI > 8 || MI < 1) continue;
        if (RB > rb2 && (S + 2 * rb2 - 1) / (2 * rb2) == MI) continue;
        for (int WN : {4, 2}) {
            Tiling t;
            t.MI = MI;
            t.WM = 2;
            t.NI = 2;
            t.WN = WN;
            t.S = S;
            t.RB = RB;
            t.MpB = 16 * MI;
            t.Mp = RB * t.MpB;
            t.Kp = Kp;
            t.BN = 16 * WN;
            t.LDX = t.BN + 4;
            t.nstage = 3;
            t.smem = sizeof(double) * static_cast<size_t>(t.nstage) * (kBK * t.LDX + t.MpB * kLDJ);
            if (t.smem > kSmemPerCTA) continue;
            int occ = 0;
            dispatch_mode(t, ModeGeom{}, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, &occ);
            t.ctas_per_sm = occ;
            if (occ < 1) continue;
            const double eff = 0.85 + 0.15 * static_cast<double>(S) / (RB * 2 * MI);
            c.emplace_back(std::min(occ * 2 * t.WN, 16) * eff + 0.02 * WN - 0.05 * RB - 0.06, t);
        }
    }
    std::stable_sort(c.begin(), c.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
    std::vector<Tiling> out;
    // the dense resident-factor kernel (dense_res.cu) measured slower than the streaming kernel on every
    // BASELINE shape (c4 modes 0.156 vs 0.118 ms, c5p5 time GEMM 9.9 vs 7.8 ms): opt-in only
    const char* dk = std::getenv("STIGA_DENSE_KERNEL");
    if (dk && std::string(dk) == "res") out = mode_res_candidates(m, n, false);
    for (auto& e : c) out.push_back(e.second);
    return out;
}

Tiling choose_mode_tiling(int m, int n, bool prescale) {
    (void)prescale;  // the D^-1/2 pre-scale is a separate elementwise pass
    const std::vector<Tiling> c = mode_tiling_candidates(m, n);
    for (const Tiling& t : c)
        if (!t.res) return t;  // untuned callers take the streaming kernel's heuristic first choice
    Tiling t;
    t.MI = 0;
    return t;
}


size_t prescale_smem(const Tiling& t) {
    return t.smem + sizeof(double) * static_cast<size_t>(t.nstage) * kBK * t.LDX;
}

bool prescale_fits(const Tiling& t) {
    if (t.res) return mode_res_smem(t, true) + 1024 <= kSmemPerCTA;
    if (t.fold == 2) return fold_res_prescale_smem(t) + 1024 <= kSmemPerCTA;
    if (t.fold) return fold_prescale_smem(t) <= kSmemPerCTA;
    return t.WM == 1 && prescale_smem(t) <= kSmemPerCTA;
}

cudaError_t launch_mode_product(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jpad,
                                const double* post_scale, cudaStream_t st, const double* pre_scale, const Scatter* sc) {
    if (g.ncols <= 0) return cudaSuccess;
    if (pre_scale && !prescale_fits(t)) return cudaErrorInvalidValue;
    if (t.res) {
        if (sc) return cudaErrorInvalidValue;  // no scatter epilogue on the resident kernel
        return launch_mode_res(t, g, X, Y, Jpad, post_scale, pre_scale, st);
    }
    if (sc && (pre_scale || post_scale || sc->G < 1 || sc->G > kMaxRanks)) return cudaErrorInvalidValue;
    return dispatch_mode(t, g, X, Y, Jpad, post_scale, pre_scale, st, nullptr, sc);
}


}  // namespace gpu
}  // namespace stiga
