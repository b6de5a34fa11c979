// Time direction of the FD apply: the time-fused kernel (fd_time_impl.cuh), its tiling candidates
// and launcher.
#include "fd_time_impl.cuh"

#include <cstdlib>
#include <string>

namespace stiga {
namespace gpu {

namespace {

cudaError_t dispatch_time(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jt,
                          const double* J, const ArrowParams& ap, cudaStream_t st, int* occ,
                          const Scatter* sc = nullptr) {
    if (sc) return dispatch_time_scatter(t, g, X, Jt, J, ap, st, occ, sc);
    return dispatch_time_v<false>(t, g, X, Y, Jt, J, ap, st, occ, nullptr);
}

}  // namespace

std::vector<Tiling> time_tiling_candidates(int nt) {
    std::vector<std::pair<double, Tiling>> c;
    int force_wm = 0, force_wn = 0, force_ns = 0;  // debugging aid: STIGA_FORCE_TIME_TILING="WM,WN,NS"
    if (const char* f = std::getenv("STIGA_FORCE_TIME_TILING"))
        std::sscanf(f, "%d,%d,%d", &force_wm, &force_wn, &force_ns);
    const int S = (nt + 7) / 8;
    const int Kp = (nt + 3) / 4 * 4;
    for (int WM : {1, 2, 3, 4}) {  // WM = 3: S = 9 (c4, c5p2) splits evenly into 3 x 3 strips
        const int MI = (S + WM - 1) / WM;
        if (MI > 13 || MI < 1) continue;
        for (int WN : {4, 2}) {
            if (WM == 4 && WN == 4) continue;
            if ((force_wm && WM != force_wm) || (force_wn && WN != force_wn)) continue;
            for (int ns : {3, 2}) {
                if (force_ns && ns != force_ns) continue;
                Tiling t;
                t.MI = MI;
                t.WM = WM;
                t.NI = 2;
                t.WN = WN;
                t.S = S;
                t.RB = 1;
                t.MpB = 8 * MI * WM;
                t.Mp = t.MpB;
                t.Kp = Kp;
                t.BN = 16 * WN;
                t.LDX = t.BN + 4;
                t.Zrows = Kp;
                t.nstage = ns;
                t.smem = sizeof(double) * (static_cast<size_t>(Kp) * t.LDX +
                                           static_cast<size_t>(ns) * (kBK * t.LDX + t.MpB * kLDJ) +
                                           7 * static_cast<size_t>(nt / 2 + 1) + 3 * static_cast<size_t>(t.BN) +
                                           (WM == 3 ? 6 * static_cast<size_t>(t.BN) : 0));
                if (t.smem > kSmemPerCTA) continue;
                int occ = 0;
                ArrowParams ap;
                dispatch_time(t, ModeGeom{}, nullptr, nullptr, nullptr, nullptr, ap, nullptr, &occ);
                t.ctas_per_sm = occ;
                if (occ < 1) continue;
                const double eff = 0.85 + 0.15 * static_cast<double>(S) / (WM * MI);
                c.emplace_back(std::min(occ * WM * WN, 16) * eff + 0.01 * ns + 0.02 * WN, t);
            }
        }
    }
    std::stable_sort(c.begin(), c.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
    std::vector<Tiling> out;
    // the resident-U_t kernel (time_res.cu) measured slower than this streaming kernel on every
    // BASELINE shape (c4 0.339 vs 0.282 ms, c3 3.48 vs 1.65 ms: the arrowhead phase leaves the DMMA
    // pipe idle with one or two CTAs per SM): opt-in only
    const char* tk = std::getenv("STIGA_TIME_KERNEL");
    if (tk && std::string(tk) == "res" && !force_wm) out = time_res_candidates(nt);
    for (auto& e : c) out.push_back(e.second);
    return out;
}

Tiling choose_time_tiling(int nt) {
    const std::vector<Tiling> c = time_tiling_candidates(nt);
    for (const Tiling& t : c)
        if (!t.res) return t;
    Tiling t;
    t.MI = 0;
    return t;
}


cudaError_t launch_time_fused(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jt_pad,
                              const double* J_pad, const ArrowParams& ap, cudaStream_t st, const Scatter* sc) {
    if (g.ncols <= 0) return cudaSuccess;
    if (sc && (sc->G < 1 || sc->G > kMaxRanks)) return cudaErrorInvalidValue;
    if (t.res == 2) {
        if (sc) return cudaErrorInvalidValue;  // no scatter epilogue on the resident kernel
        return launch_time_res(t, g, X, Y, J_pad, ap, st);
    }
    return dispatch_time(t, g, X, Y, Jt_pad, J_pad, ap, st, nullptr, sc);
}


}  // namespace gpu
}  // namespace stiga
