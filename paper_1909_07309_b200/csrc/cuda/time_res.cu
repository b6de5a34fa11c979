// Time direction of the FD apply (U_t^T -> block-arrowhead solve -> U_t, fdsolve.cpp:159-161 with
// arrowhead_solve fdsolve.cpp:24-65) with U_t RESIDENT in shared memory and persistent CTAs
// (Tiling::res == 2), for the short time factors of configs c4 / c5p2 (n_t <= ~70):
//  * one copy of U_t serves both products: U_t^T fragments are read transposed from the same rows
//    (row stride == 4 mod 16 doubles keeps both access patterns bank-conflict free), so a CTA needs
//    ~48 KB for the factor and two CTAs share an SM -- one CTA's arrowhead phase (FP64 CUDA-core
//    work, no DMMA) overlaps the other CTA's products;
//  * a producer warp streams the 16-row fiber chunks of the U_t^T product into an NS-deep ring (full /
//    empty mbarriers) across tiles; the U_t product takes its B operand from the resident Z tile;
//  * consumer warps (two per sub-partition with two CTAs per SM) own strip groups x fiber groups; they
//    synchronise among themselves with a named barrier (the producer never waits on them), and
//    issue only unpredicated MMAs (padded rows / columns of U_t are zeros in smem).
#include "fd_common.cuh"
#include "res_common.cuh"

#include <algorithm>
#include <vector>

namespace stiga {
namespace gpu {

namespace {

using namespace resdev;

struct TArgs {
    ModeGeom geo;
    int Kp, LDA, KR, NQ, S, Mp;  // KR: resident rows (= cols) of U_t, max(8 S, Kp); Mp: rows of the global U_t
    long long ntiles;
};

template <int NI, int WF>
struct TShape {
    static constexpr int BN = 8 * NI * WF;
    static constexpr int LDX = BN + 4;
    static constexpr int XB = kBK * LDX;
    static constexpr int FPL = (BN + 31) / 32;
};

__device__ __forceinline__ void consumer_sync(int nthreads) {
    asm volatile("bar.sync 1, %0;\n" ::"r"(nthreads) : "memory");
}

// One 16-deep chunk of acc += A B: A element (strip mi, k-step kk) at a[mi * sm + kk * 4 * sk] (TRANS:
// U_t^T read from U_t), B fragments at b[kk * 4 * LDX + ni * 8]; fragments double-buffered.
template <int MSW, int NI, int LDX, int KS>
__device__ __forceinline__ void tchunk(const double* __restrict__ a, int sm, int sk, const double* __restrict__ b,
                                       double (&c)[MSW][NI][2]) {
    double av[2][MSW], bv[2][NI];
#pragma unroll
    for (int mi = 0; mi < MSW; ++mi) av[0][mi] = a[mi * sm];
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) bv[0][ni] = b[ni * 8];
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
        const int cur = kk & 1, nxt = cur ^ 1;
        if (kk + 1 < KS) {
#pragma unroll
            for (int mi = 0; mi < MSW; ++mi) av[nxt][mi] = a[mi * sm + (kk + 1) * 4 * sk];
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) bv[nxt][ni] = b[(kk + 1) * 4 * LDX + ni * 8];
        }
#pragma unroll
        for (int mi = 0; mi < MSW; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) rdmma(c[mi][ni][0], c[mi][ni][1], av[cur][mi], bv[cur][ni]);
    }
}

template <int MSW, int NI, int LDX>
__device__ __forceinline__ void tchunk_ks(int ks, const double* a, int sm, int sk, const double* b,
                                          double (&c)[MSW][NI][2]) {
    if (ks == 4) tchunk<MSW, NI, LDX, 4>(a, sm, sk, b, c);
    else if (ks == 3) tchunk<MSW, NI, LDX, 3>(a, sm, sk, b, c);
    else if (ks == 2) tchunk<MSW, NI, LDX, 2>(a, sm, sk, b, c);
    else tchunk<MSW, NI, LDX, 1>(a, sm, sk, b, c);
}

// Block-arrowhead solve of the resident Z tile (same arithmetic as arrowhead_tile in fd_common.cuh):
// NT consumer threads, P = NT / BN per column.
template <int NT, int BN, int LDX>
__device__ __forceinline__ void arrow_res(double* Zs, const ArrowParams& ap, const double* cs, const double* ccol) {
    const int NP = arrow_np(ap);
    constexpr int P = NT / BN;
    static_assert(P >= 1 && P <= 32 && (P & (P - 1)) == 0, "threads per column must be a power of two <= 32");
    const int tid = threadIdx.x;
    const int c = tid / P;
    const int p = tid - c * P;
    const double lam = ccol[c], linv = ccol[BN + c];
    const double nu = ap.nu, inv_nu = ap.inv_nu, gam = ap.gamma;
    const double nulam = nu * lam;
    const int nt = ap.n_t;
    double* col = Zs + c;
    const double slast = col[(nt - 1) * LDX];
    double part = 0.0;
    for (int j = p; j < ap.npairs; j += P) {
        double xa, xb;
        const double rinv = pair_rinv(nulam, linv, cs[j]);
        pair_apply(rinv, linv, inv_nu, cs[NP + j], cs[2 * NP + j], col[(2 * j) * LDX], col[(2 * j + 1) * LDX], xa, xb);
        part = fma(cs[5 * NP + j], xa, fma(cs[6 * NP + j], xb, part));
    }
    double xz = 0.0;
    if (ap.zero_count && p == 0) {
        xz = linv * col[(nt - 2) * LDX] * inv_nu;
        part += gam * __ldg(ap.g + nt - 2) * xz;
    }
#pragma unroll
    for (int off = P >> 1; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
    const double xlast = ccol[2 * BN + c] * (slast + part);
    for (int j = p; j < ap.npairs; j += P) {
        double xa, xb;
        const double rinv = pair_rinv(nulam, linv, cs[j]);
        const double u = fma(-cs[5 * NP + j], xlast, col[(2 * j) * LDX]);
        const double w = fma(-cs[6 * NP + j], xlast, col[(2 * j + 1) * LDX]);
        pair_apply(rinv, linv, inv_nu, cs[NP + j], cs[2 * NP + j], u, w, xa, xb);
        col[(2 * j) * LDX] = xa;
        col[(2 * j + 1) * LDX] = xb;
    }
    if (p == 0) {
        if (ap.zero_count) col[(nt - 2) * LDX] = xz - (gam * __ldg(ap.g + nt - 2) * inv_nu) * (linv * xlast);
        col[(nt - 1) * LDX] = xlast;
    }
}

template <int MSW, int NI, int WS, int WF, int NS>
__global__ void __launch_bounds__(32 * (WS * WF + 1), 2)
    time_res_kernel(TArgs a, const double* __restrict__ X, double* __restrict__ Y, const double* __restrict__ J,
                    ArrowParams ap) {
    constexpr int NW = WS * WF, NT = 32 * NW;
    using SH = TShape<NI, WF>;
    extern __shared__ __align__(16) double smem[];
    __shared__ uint64_t full[NS], empty[NS];
    const int LDA = a.LDA, KR = a.KR;
    double* sA = smem;                                         // [KR][LDA] U_t, zero padded
    double* Zs = sA + static_cast<size_t>(KR) * LDA;           // [Kp][LDX] resident Z tile
    double* sX = Zs + static_cast<size_t>(a.Kp) * SH::LDX;     // [NS][XB] fiber chunks
    double* cs = sX + NS * SH::XB;                             // 7 x NP pair constants
    double* ccol = cs + 7 * arrow_np(ap);                      // 3 x BN column constants
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    for (int i = tid; i < KR * LDA; i += blockDim.x) {
        const int row = i / LDA, col = i - row * LDA;
        sA[i] = (row < a.Mp && col < a.Kp) ? J[static_cast<long long>(row) * a.Kp + col] : 0.0;
    }
    stage_arrow_consts(ap, cs);
    if (tid == 0) {
        for (int s = 0; s < NS; ++s) {
            rmb_init(&full[s], 32);
            rmb_init(&empty[s], NW);
        }
    }
    __syncthreads();

    const long long L = a.geo.L, ncols = a.geo.ncols;
    const int n = a.geo.n;
    if (warp == NW) {
        // ---------------- producer warp: the U_t^T product's fiber chunks ----------------
        unsigned seq = 0;
        for (long long tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
            const long long c0 = tile * SH::BN;
            const double* fp0[SH::FPL];
            bool fv[SH::FPL];
#pragma unroll
            for (int u = 0; u < SH::FPL; ++u) {
                const long long cc = c0 + lane + 32 * u;
                fv[u] = cc < ncols && lane + 32 * u < SH::BN;
                const long long r = (fv[u] ? cc : 0) / L;
                fp0[u] = X + ((fv[u] ? cc : 0) - r * L) + L * static_cast<long long>(n) * r;
            }
            for (int q = 0; q < a.NQ; ++q, ++seq) {
                const int s = seq % NS;
                rmb_wait(&empty[s], ((seq / NS) & 1u) ^ 1u);
                const unsigned sa = ru32(sX + s * SH::XB);
                const int ra0 = q * kBK;
#pragma unroll
                for (int u = 0; u < SH::FPL; ++u) {
                    if (SH::BN % 32 != 0 && lane + 32 * u >= SH::BN) continue;
                    const double* pa = fp0[u] + L * ra0;
                    unsigned da = sa + 8u * (lane + 32 * u);
                    for (int r = 0; r < kBK; ++r) {
                        const bool va = fv[u] && ra0 + r < n;
                        rcp8(da, va ? pa : X, va);
                        pa += L;
                        da += 8u * SH::LDX;
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
    const int fcol = wf * NI * 8 + g;
    const double* aT = sA + t * LDA + so * 8 + g;   // U_t^T (row r, k) = U_t (k, r)
    const double* aN = sA + (so * 8 + g) * LDA + t;  // U_t (row r, k)
    unsigned seq = 0;
    for (long long tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
        const long long c0 = tile * SH::BN;
        double c[MSW][NI][2];
#pragma unroll
        for (int mi = 0; mi < MSW; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) c[mi][ni][0] = c[mi][ni][1] = 0.0;
        // Z = U_t^T X (fdsolve.cpp:159, the forward time factor)
        for (int q = 0; q < a.NQ; ++q, ++seq) {
            const int s = seq % NS;
            rmb_wait(&full[s], (seq / NS) & 1u);
            const int k0 = q * kBK;
            tchunk_ks<MSW, NI, SH::LDX>(min(kBK, a.Kp - k0) >> 2, aT + k0 * LDA, 8, LDA,
                                        sX + s * SH::XB + t * SH::LDX + fcol, c);
            __syncwarp();
            if (lane == 0) rmb_arrive(&empty[s]);
        }
        consumer_sync(NT);  // every consumer is done reading the previous tile's Z and column constants
        stage_column_consts(ap, c0, ncols, SH::BN, ccol);
#pragma unroll
        for (int mi = 0; mi < MSW; ++mi) {
            const int row = (so + mi) * 8 + g;
            if (row < a.Kp) {
#pragma unroll
                for (int ni = 0; ni < NI; ++ni) {
                    const int col = (wf * NI + ni) * 8 + 2 * t;
                    Zs[row * SH::LDX + col] = c[mi][ni][0];
                    Zs[row * SH::LDX + col + 1] = c[mi][ni][1];
                }
            }
        }
        consumer_sync(NT);
        if (!(ap.debug & 1)) arrow_res<NT, SH::BN, SH::LDX>(Zs, ap, cs, ccol);
        consumer_sync(NT);
        // y = U_t z (fdsolve.cpp:161)
#pragma unroll
        for (int mi = 0; mi < MSW; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) c[mi][ni][0] = c[mi][ni][1] = 0.0;
        for (int q = 0; q < a.NQ; ++q) {
            const int k0 = q * kBK;
            tchunk_ks<MSW, NI, SH::LDX>(min(kBK, a.Kp - k0) >> 2, aN + k0, 8 * LDA, 1,
                                        Zs + (k0 + t) * SH::LDX + fcol, c);
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
                ob[ni][v] = ((cv[ni][v] ? cc : 0) - r * L) + L * static_cast<long long>(n) * r;
            }
#pragma unroll
        for (int mi = 0; mi < MSW; ++mi) {
            const int i = (so + mi) * 8 + g;
            if (i >= n) continue;
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                for (int v = 0; v < 2; ++v)
                    if (cv[ni][v]) Y[ob[ni][v] + L * i] = c[mi][ni][v];
        }
    }
}

int tlda_of(int cols) { return cols + ((4 - cols % 16) % 16 + 16) % 16; }

size_t tres_smem(int KR, int Kp, int NI, int WF, int NS, int n_t) {
    const int BN = 8 * NI * WF, LDX = BN + 4;
    return sizeof(double) * (static_cast<size_t>(KR) * tlda_of(KR) + static_cast<size_t>(Kp) * LDX +
                             static_cast<size_t>(NS) * kBK * LDX + 7 * (n_t / 2 + 1) + 3 * BN);
}

int g_tsms = 0;

template <int MSW, int NI, int WS, int WF, int NS>
cudaError_t tres_launch_t(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                          const ArrowParams& ap, cudaStream_t st, int* occ) {
    auto k = time_res_kernel<MSW, NI, WS, WF, NS>;
    const int KR = std::max(8 * t.S, t.Kp);
    const size_t smem = tres_smem(KR, t.Kp, NI, WF, NS, g.n);
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) {
        cudaGetLastError();
        if (occ) *occ = 0;
        return occ ? cudaSuccess : e;
    }
    if (occ) {
        int nb = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, 32 * (WS * WF + 1), smem) != cudaSuccess) {
            cudaGetLastError();
            nb = 0;
        }
        *occ = nb;
        return cudaSuccess;
    }
    if (g_tsms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_tsms, cudaDevAttrMultiProcessorCount, dev);
        if (g_tsms <= 0) g_tsms = 148;
    }
    TArgs a;
    a.geo = g;
    a.Kp = t.Kp;
    a.KR = KR;
    a.LDA = tlda_of(KR);
    a.NQ = (t.Kp + kBK - 1) / kBK;
    a.S = t.S;
    a.Mp = t.Mp;
    a.ntiles = (g.ncols + t.BN - 1) / t.BN;
    const long long grid = std::min<long long>(a.ntiles, static_cast<long long>(g_tsms) * std::max(1, t.ctas_per_sm));
    k<<<static_cast<unsigned>(grid), 32 * (WS * WF + 1), smem, st>>>(a, X, Y, J, ap);
    return cudaGetLastError();
}

cudaError_t tres_dispatch(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                          const ArrowParams& ap, cudaStream_t st, int* occ) {
#define STIGA_TRES(A_, B_, C_, D_, E_)                                                          \
    if (t.MI == A_ && t.NI == B_ && t.WM == C_ && t.WN == D_ && t.nstage == E_)                \
        return tres_launch_t<A_, B_, C_, D_, E_>(t, g, X, Y, J, ap, st, occ);
    STIGA_TRES(9, 1, 1, 4, 4)   // n_t <= 72: 4 consumer warps, 32 fibers
    STIGA_TRES(9, 2, 1, 2, 4)   // n_t <= 72: 2 consumer warps x 2 fiber groups
    STIGA_TRES(5, 1, 2, 2, 4)   // n_t <= 80: 2 strip groups x 2 fiber groups
    STIGA_TRES(5, 2, 2, 2, 4)   // n_t <= 80, 32 fibers
    STIGA_TRES(7, 1, 2, 2, 3)   // n_t <= 112
#undef STIGA_TRES
    return cudaErrorInvalidValue;
}

}  // namespace

std::vector<Tiling> time_res_candidates(int n_t) {
    std::vector<Tiling> out;
    const int S = (n_t + 7) / 8;
    const int Kp = (n_t + 3) / 4 * 4;
    const int shapes[5][5] = {{9, 1, 1, 4, 4}, {9, 2, 1, 2, 4}, {5, 1, 2, 2, 4}, {5, 2, 2, 2, 4}, {7, 1, 2, 2, 3}};
    for (const auto& sh : shapes) {
        const int cover = sh[0] * sh[2];
        if (cover < S || cover > S + 1) continue;  // strips must cover n_t with at most one padded strip
        Tiling t;
        t.res = 2;
        t.MI = sh[0];
        t.NI = sh[1];
        t.WM = sh[2];
        t.WN = sh[3];
        t.nstage = sh[4];
        t.S = S;
        t.RB = 1;
        t.Kp = Kp;
        t.BN = 8 * t.NI * t.WN;
        t.LDX = t.BN + 4;
        t.Zrows = Kp;
        t.MpB = 8 * S;
        t.Mp = 8 * S;
        int occ = 0;
        tres_dispatch(t, ModeGeom{1, 1, n_t, n_t}, nullptr, nullptr, nullptr, ArrowParams{}, nullptr, &occ);
        if (occ < 1) continue;
        t.ctas_per_sm = std::min(occ, 2);
        t.smem = tres_smem(std::max(8 * S, Kp), Kp, t.NI, t.WN, t.nstage, n_t);
        out.push_back(t);
    }
    return out;
}

cudaError_t launch_time_res(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J,
                            const ArrowParams& ap, cudaStream_t st) {
    if (g.ncols <= 0) return cudaSuccess;
    if (t.res != 2 || g.m != g.n) return cudaErrorInvalidValue;
    return tres_dispatch(t, g, X, Y, J, ap, st, nullptr);
}

}  // namespace gpu
}  // namespace stiga
