// Dense mode product Y = (I (x) J (x) I) X (mode_product, kronop.cpp:43-73) with a row block of the
// factor RESIDENT in shared memory, persistent CTAs and a warp-specialised cp.async -> mbarrier
// pipeline (Tiling::res == 1) -- the dense counterpart of fold_res.cu, for the directions that are not
// mirror symmetric (the deformed cube of config 4, the time factors U_t^T / U_t):
//  * CTA b owns row block rb = b % RB (8 MS rows of J, <= ~120 KB) for the whole launch and walks the
//    fiber tiles b / RB, b / RB + grid / RB, ...; the RB CTAs of one tile run side by side, so the
//    tile's fiber data is read from HBM once and from L2 by the other row blocks;
//  * one producer warp streams 16-row fiber chunks (+ the matching D^-1/2 chunk for the fused
//    pre-scale) with 8-byte cp.async into an NS-deep ring (full / empty mbarriers), across tiles;
//  * consumer warps: WS strip groups x WF fiber groups, MSW strips x NI 8-fiber groups each, two per
//    SM sub-partition (a warp issues at most one DMMA.8x8x4 per ~16 cycles), no predicated MMAs
//    (padded strips are zero rows), fragments double-buffered, register epilogue (+ D^-1/2 post-scale).
#include "fd_kernels.cuh"
#include "res_common.cuh"

#include <algorithm>
#include <cstdint>
#include <vector>

namespace stiga {
namespace gpu {

namespace {

using namespace resdev;

constexpr int kBK = 16;
constexpr size_t kSmemPerCTA = 227 * 1024;

struct DArgs {
    ModeGeom geo;
    int Kp, LDA, NQ, RB, Mp;  // Mp: rows of the padded global factor
    long long ntiles;
};

template <int NI, int WF, bool PS>
struct DShape {
    static constexpr int BN = 8 * NI * WF;
    static constexpr int LDX = BN + 4;
    static constexpr int XB = kBK * LDX;
    static constexpr int STAGE = XB * (PS ? 2 : 1);  // fiber chunk [+ D^-1/2 chunk]
    static constexpr int FPL = (BN + 31) / 32;
};

template <int MSW, int NI, int WF, bool PS>
__device__ __forceinline__ void dfrag(const double* __restrict__ a1, const double* __restrict__ xa, int LDA, int kk,
                                      double (&av)[MSW], double (&b)[NI]) {
    using SH = DShape<NI, WF, PS>;
#pragma unroll
    for (int mi = 0; mi < MSW; ++mi) av[mi] = a1[mi * 8 * LDA + kk * 4];
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
        b[ni] = xa[kk * 4 * SH::LDX + ni * 8];
        if (PS) b[ni] *= xa[SH::XB + kk * 4 * SH::LDX + ni * 8];
    }
}

template <int MSW, int NI, int WF, bool PS, int KS>
__device__ __forceinline__ void dchunk(const double* __restrict__ a1, const double* __restrict__ xa, int LDA,
                                       double (&c)[MSW][NI][2]) {
    double av[2][MSW], b[2][NI];
    dfrag<MSW, NI, WF, PS>(a1, xa, LDA, 0, av[0], b[0]);
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
        const int cur = kk & 1, nxt = cur ^ 1;
        if (kk + 1 < KS) dfrag<MSW, NI, WF, PS>(a1, xa, LDA, kk + 1, av[nxt], b[nxt]);
#pragma unroll
        for (int mi = 0; mi < MSW; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) rdmma(c[mi][ni][0], c[mi][ni][1], av[cur][mi], b[cur][ni]);
    }
}

template <int MSW, int NI, int WS, int WF, int NS, bool POST, bool PS>
__global__ void __launch_bounds__(32 * (WS * WF + 1), 1)
    dense_res_kernel(DArgs a, const double* __restrict__ X, double* __restrict__ Y, const double* __restrict__ J,
                     const double* __restrict__ post, const double* __restrict__ pre) {
    constexpr int NW = WS * WF;
    constexpr int MR = 8 * MSW * WS;  // resident rows of this CTA's row block
    using SH = DShape<NI, WF, PS>;
    extern __shared__ __align__(16) double smem[];
    __shared__ uint64_t full[NS], empty[NS];
    const int LDA = a.LDA;
    double* sA = smem;               // [MR][LDA]
    double* sX = smem + MR * LDA;    // [NS][STAGE]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rb = blockIdx.x % a.RB;
    const int row0 = rb * MR;
    const long long tstride = gridDim.x / a.RB;

    for (int i = tid; i < MR * a.Kp; i += blockDim.x) {
        const int row = i / a.Kp, col = i - row * a.Kp;
        const int gr = row0 + row;
        sA[row * LDA + col] = gr < a.Mp ? J[static_cast<long long>(gr) * a.Kp + col] : 0.0;
    }
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            rmb_init(&full[s], 32);
            rmb_init(&empty[s], NW);
        }
    }
    __syncthreads();

    const long long L = a.geo.L, ncols = a.geo.ncols;
    const int n = a.geo.n, m = a.geo.m;
    if (warp == NW) {
        // ---------------- producer warp ----------------
        unsigned seq = 0;
        for (long long tile = blockIdx.x / a.RB; tile < a.ntiles; tile += tstride) {
            const long long c0 = tile * SH::BN;
            const bool full_tile = c0 + SH::BN <= ncols;
            const double* fp0[SH::FPL];
            bool fv[SH::FPL];
            if (L != 1) {
#pragma unroll
                for (int u = 0; u < SH::FPL; ++u) {
                    const long long cc = c0 + lane + 32 * u;
                    fv[u] = cc < ncols && lane + 32 * u < SH::BN;
                    const long long r = (fv[u] ? cc : 0) / L;
                    fp0[u] = X + ((fv[u] ? cc : 0) - r * L) + L * static_cast<long long>(n) * r;
                }
            }
            const int r16 = lane & 15, fpar = lane >> 4;
            const double* f1 = X + (full_tile || c0 + fpar < ncols ? c0 + fpar : 0) * n;
            const long long dofs = PS ? pre - X : 0;
            for (int q = 0; q < a.NQ; ++q, ++seq) {
                const int s = seq % NS;
                rmb_wait(&empty[s], ((seq / NS) & 1u) ^ 1u);
                const unsigned sa = ru32(sX + s * SH::STAGE);
                const int ra0 = q * kBK;
                const bool rows_in = ra0 + kBK <= n;
                if (L == 1) {
                    const int rowa = ra0 + r16;
                    const double* pa = f1 + rowa;
                    const long long step = 2LL * n;
                    unsigned da = sa + 8u * (r16 * SH::LDX + fpar);
                    const bool va = rowa < n;
                    for (int f = 0; f < SH::BN; f += 2) {
                        const bool ok = (full_tile && rows_in) || (va && c0 + fpar + f < ncols);
                        rcp8(da, ok ? pa : X, ok);
                        if (PS) rcp8(da + 8u * SH::XB, ok ? pa + dofs : X, ok);
                        pa += step;
                        da += 16u;
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < SH::FPL; ++u) {
                        if (SH::BN % 32 != 0 && lane + 32 * u >= SH::BN) continue;
                        const double* pa = fp0[u] + L * ra0;
                        unsigned da = sa + 8u * (lane + 32 * u);
                        if (fv[u] && rows_in) {
#pragma unroll 8
                            for (int r = 0; r < kBK; ++r) {
                                rcp8(da, pa, true);
                                if (PS) rcp8(da + 8u * SH::XB, pa + dofs, true);
                                pa += L;
                                da += 8u * SH::LDX;
                            }
                        } else {
                            for (int r = 0; r < kBK; ++r) {
                                const bool va = fv[u] && ra0 + r < n;
                                rcp8(da, va ? pa : X, va);
                                if (PS) rcp8(da + 8u * SH::XB, va ? pa + dofs : X, va);
                                pa += L;
                                da += 8u * SH::LDX;
                            }
                        }
                    }
                }
                rmb_cp_arrive(&full[s]);
            }
        }
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        return;
    }

    // ---------------- consumer warps ----------------
    const int g = lane >> 2, t = lane & 3;
    const int ws = warp / WF, wf = warp - ws * WF;
    const int so = ws * MSW;
    const double* a1 = sA + (so * 8 + g) * LDA + t;
    const int fcol = wf * NI * 8 + g;
    unsigned seq = 0;
    for (long long tile = blockIdx.x / a.RB; tile < a.ntiles; tile += tstride) {
        const long long c0 = tile * SH::BN;
        double c[MSW][NI][2];
#pragma unroll
        for (int mi = 0; mi < MSW; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) c[mi][ni][0] = c[mi][ni][1] = 0.0;
        for (int q = 0; q < a.NQ; ++q, ++seq) {
            const int s = seq % NS;
            rmb_wait(&full[s], (seq / NS) & 1u);
            const double* xa = sX + s * SH::STAGE + t * SH::LDX + fcol;
            const int k0 = q * kBK;
            const int ks = min(kBK, a.Kp - k0) >> 2;
            if (ks == 4) dchunk<MSW, NI, WF, PS, 4>(a1 + k0, xa, LDA, c);
            else if (ks == 3) dchunk<MSW, NI, WF, PS, 3>(a1 + k0, xa, LDA, c);
            else if (ks == 2) dchunk<MSW, NI, WF, PS, 2>(a1 + k0, xa, LDA, c);
            else dchunk<MSW, NI, WF, PS, 1>(a1 + k0, xa, LDA, c);
            __syncwarp();
            if (lane == 0) rmb_arrive(&empty[s]);
        }
        long long ob[NI][2];
        bool cv[NI][2];
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const long long cc = c0 + (wf * NI + ni) * 8 + 2 * t + v;
                cv[ni][v] = cc < ncols;
                const long long r = (cv[ni][v] ? cc : 0) / L;
                ob[ni][v] = ((cv[ni][v] ? cc : 0) - r * L) + L * static_cast<long long>(m) * r;
            }
        double sc[MSW][NI][2];
        if constexpr (POST) {  // every scale value loaded before the first store
#pragma unroll
            for (int mi = 0; mi < MSW; ++mi) {
                const int i = row0 + (so + mi) * 8 + g;
#pragma unroll
                for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                    for (int v = 0; v < 2; ++v)
                        sc[mi][ni][v] = (cv[ni][v] && i < m) ? __ldg(post + ob[ni][v] + L * i) : 0.0;
            }
        }
#pragma unroll
        for (int mi = 0; mi < MSW; ++mi) {
            const int i = row0 + (so + mi) * 8 + g;
            if (i >= m) continue;
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                for (int v = 0; v < 2; ++v)
                    if (cv[ni][v]) Y[ob[ni][v] + L * i] = POST ? sc[mi][ni][v] * c[mi][ni][v] : c[mi][ni][v];
        }
    }
}

int dlda_of(int Kp) { return Kp + ((4 - Kp % 16) % 16 + 16) % 16; }

size_t dres_smem(int MR, int NI, int WF, int NS, int Kp, bool ps) {
    const int BN = 8 * NI * WF;
    return sizeof(double) * (static_cast<size_t>(MR) * dlda_of(Kp) + static_cast<size_t>(NS) * kBK * (BN + 4) * (ps ? 2 : 1));
}

int g_dsms = 0;

template <int MSW, int NI, int WS, int WF, int NS>
cudaError_t dres_launch_t(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                          const double* post, const double* pre, cudaStream_t st, int* occ) {
    constexpr int NW = WS * WF;
    auto k = pre ? dense_res_kernel<MSW, NI, WS, WF, NS, false, true>
                 : (post ? dense_res_kernel<MSW, NI, WS, WF, NS, true, false>
                         : dense_res_kernel<MSW, NI, WS, WF, NS, false, false>);
    const size_t smem = dres_smem(8 * MSW * WS, NI, WF, NS, t.Kp, pre != nullptr);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) {
        cudaGetLastError();
        if (occ) *occ = 0;
        return occ ? cudaSuccess : e;
    }
    if (occ) {
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 32 * (NW + 1), smem) != cudaSuccess) {
            cudaGetLastError();
            nb = 0;
        }
        *occ = nb;
        return cudaSuccess;
    }
    if (g_dsms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_dsms, cudaDevAttrMultiProcessorCount, dev);
        if (g_dsms <= 0) g_dsms = 148;
    }
    DArgs a;
    a.geo = g;
    a.Kp = t.Kp;
    a.LDA = dlda_of(t.Kp);
    a.NQ = (t.Kp + kBK - 1) / kBK;
    a.RB = t.RB;
    a.Mp = t.Mp;
    a.ntiles = (g.ncols + t.BN - 1) / t.BN;
    const long long per_rb = std::max<long long>(1, std::min<long long>(a.ntiles, g_dsms / t.RB));
    const long long grid = per_rb * t.RB;
    k<<<static_cast<unsigned>(grid), 32 * (NW + 1), smem, st>>>(a, X, Y, J, post, pre);
    return cudaGetLastError();
}

// Tiling fields: MI = strips per warp (MSW), WM = strip groups (WS), WN = fiber groups (WF), NI, nstage.
cudaError_t dres_dispatch(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                          const double* post, const double* pre, cudaStream_t st, int* occ) {
#define STIGA_DRES(A_, B_, C_, D_, E_)                                                          \
    if (t.MI == A_ && t.NI == B_ && t.WM == C_ && t.WN == D_ && t.nstage == E_)                \
        return dres_launch_t<A_, B_, C_, D_, E_>(t, g, X, Y, J, post, pre, st, occ);
    STIGA_DRES(11, 1, 1, 8, 4)
    STIGA_DRES(9, 1, 1, 8, 4)
    STIGA_DRES(9, 2, 1, 4, 4)
    STIGA_DRES(7, 1, 1, 8, 4)
    STIGA_DRES(5, 1, 2, 4, 4)
    STIGA_DRES(6, 1, 2, 4, 4)
    STIGA_DRES(5, 2, 2, 4, 4)
    STIGA_DRES(11, 2, 1, 4, 4)
#undef STIGA_DRES
    return cudaErrorInvalidValue;
}

}  // namespace

std::vector<Tiling> mode_res_candidates(int m, int n, bool prescale) {
    std::vector<Tiling> out;
    const int S = (m + 7) / 8;
    const int Kp = (n + 3) / 4 * 4;
    // (MSW, NI, WS, WF, NS) shapes compiled in dres_dispatch; RB row blocks cover the S strips
    const int shapes[8][5] = {{11, 1, 1, 8, 4}, {9, 1, 1, 8, 4}, {9, 2, 1, 4, 4}, {7, 1, 1, 8, 4},
                              {5, 1, 2, 4, 4}, {6, 1, 2, 4, 4}, {5, 2, 2, 4, 4}, {11, 2, 1, 4, 4}};
    for (const auto& sh : shapes) {
        const int per = sh[0] * sh[2];  // strips per row block
        const int RB = (S + per - 1) / per;
        if (RB > 3 || (RB > 1 && per * (RB - 1) >= S)) continue;
        if (per > S + 1 && RB == 1 && sh[2] == 2) continue;  // a whole idle strip group
        Tiling t;
        t.res = 1;
        t.MI = sh[0];
        t.NI = sh[1];
        t.WM = sh[2];
        t.WN = sh[3];
        t.nstage = sh[4];
        t.S = S;
        t.RB = RB;
        t.MpB = 8 * per;
        t.Mp = RB * t.MpB;
        t.Kp = Kp;
        t.BN = 8 * t.NI * t.WN;
        t.LDX = t.BN + 4;
        t.smem = dres_smem(t.MpB, t.NI, t.WN, t.nstage, Kp, prescale);
        if (t.smem + 1024 > kSmemPerCTA) continue;
        int occ = 0;
        dres_dispatch(t, ModeGeom{}, nullptr, nullptr, nullptr, nullptr, prescale ? reinterpret_cast<const double*>(8) : nullptr,
                      nullptr, &occ);
        if (occ < 1) continue;
        t.ctas_per_sm = 1;
        out.push_back(t);
    }
    return out;
}

size_t mode_res_smem(const Tiling& t, bool prescale) {
    return dres_smem(t.MpB, t.NI, t.WN, t.nstage, t.Kp, prescale);
}

cudaError_t launch_mode_res(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                            const double* post, const double* pre, cudaStream_t st) {
    if (g.ncols <= 0) return cudaSuccess;
    if (!t.res) return cudaErrorInvalidValue;
    return dres_dispatch(t, g, X, Y, J, post, pre, st, nullptr);
}

}  // namespace gpu
}  // namespace stiga
