// Folded (centrosymmetric) mode product with the factor pair RESIDENT in shared memory, a persistent
// CTA per SM and a warp-specialised cp.async -> mbarrier pipeline (Tiling::fold == 2).
//
// Same arithmetic as fold_kernels.cu (the split-basis fold of DESIGN.md §3.4 / §5; mode_product,
// kronop.cpp:43-73, on half the FLOPs):
//   forward  y[r] = sum_k A_e[r][k] (x[k] + x[n-1-k]),  y[F+r] = sum_k A_o[r][k] (x[k] - x[n-1-k])
//   backward p = A_p y_e, q = A_q y_o,  x[i] = p[i] + q[i],  x[n-1-i] = p[i] - q[i],  x[h] = p[h]
// but organised for the B200 instead of per-tile streaming of the factors:
//  * the two folded F x F factors (<= 120 KB for n <= 170) are copied into shared memory ONCE per CTA;
//    only the fiber data streams (16 B/DoF of HBM per pass, no factor traffic from L2);
//  * one CTA per SM walks the fiber tiles of the whole tensor (static stride), and one producer warp
//    keeps an NS-deep ring of 16-row fiber chunks (a chunk and its mirror / second half) in flight
//    ACROSS tile boundaries, so the next tile's first chunks land while the current tile finishes --
//    the per-tile prologue/epilogue that held the streaming kernel at 50-60 % of the DMMA pipe;
//  * the stages are filled with 8-byte cp.async (the odd tensor strides of these configurations are
//    not TMA-legal) whose completion is signalled to a full mbarrier by cp.async.mbarrier.arrive;
//    consumers release a stage through an empty mbarrier -- no CTA-wide barrier in the main loop;
//  * every consumer warp owns NI 8-fiber groups x all strips of BOTH folded matrices, so the fold
//    (x_k +- x_{n-1-k}) is formed once per B fragment and the backward combination x = p +- q is done
//    in registers;
//  * DMMA.8x8x4 (FP64 tensor core) with A fragments from the resident factors (row stride == 4 mod 16
//    doubles) and B fragments from the stage (row stride BN + 4): bank-conflict free.
#include "fd_kernels.cuh"
#include "res_common.cuh"

#include <algorithm>
#include <cstdint>
#include <vector>

namespace stiga {
namespace gpu {

namespace {

constexpr int kBK = 16;
constexpr size_t kSmemPerCTA = 227 * 1024;

using namespace resdev;

struct RArgs {
    ModeGeom geo;
    int F, h;       // folded lengths (F = h + n mod 2)
    int Kp, LDA;    // contraction length of both folded matrices (round4(F)); smem row stride (== 4 mod 16)
    int NQ;         // 16-column chunks per tile
    int S1, S2;     // live 8-row strips of the first / second matrix
    long long A2;   // offset of the second matrix in the global factor buffer (Mp * Kp)
    int Mp;         // rows of each matrix in the global factor buffer
    long long ntiles;
};

template <int NI, int NW, bool PS = false>  // NW = fiber-group warps (WF)
struct RShape {
    static constexpr int BN = 8 * NI * NW;   // fibers per tile
    static constexpr int LDX = BN + 4;       // == 4 mod 16 doubles
    static constexpr int XB = kBK * LDX;     // one 16-row chunk
    static constexpr int DOFF = 2 * XB;      // PS: the D^-1/2 chunks of both, same layout
    static constexpr int STAGE = 2 * XB * (PS ? 2 : 1);  // chunk + mirror (forward) / + second half (backward)
    static constexpr int FPL = (BN + 31) / 32;  // fibers per producer lane (L > 1)
};

// Fragments of k-step kk: A of both matrices (this warp's strips), B of both (forward: the fold).
template <int MS, int NI, int NW, bool FWD, bool PS = false>
__device__ __forceinline__ void rfrag(const double* __restrict__ a1, const double* __restrict__ a2,
                                      const double* __restrict__ xa, const double* __restrict__ xb, int LDA, int kk,
                                      double (&av1)[MS], double (&av2)[MS], double (&b1)[NI], double (&b2)[NI]) {
    using SH = RShape<NI, NW, PS>;
#pragma unroll
    for (int mi = 0; mi < MS; ++mi) {
        av1[mi] = a1[mi * 8 * LDA + kk * 4];
        av2[mi] = a2[mi * 8 * LDA + kk * 4];
    }
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
        double u = xa[kk * 4 * SH::LDX + ni * 8];
        if (PS) u *= xa[SH::DOFF + kk * 4 * SH::LDX + ni * 8];  // fused D^-1/2 pre-scale
        if (FWD) {  // xb points at the mirrored row of k-step 0; rows run backwards
            double w = xb[-kk * 4 * SH::LDX + ni * 8];
            if (PS) w *= xb[SH::DOFF - kk * 4 * SH::LDX + ni * 8];
            b1[ni] = u + w;
            b2[ni] = u - w;
        } else {
            b1[ni] = u;
            b2[ni] = xb[kk * 4 * SH::LDX + ni * 8];
        }
    }
}

// One 16-column chunk: KS k-steps of 4 over both matrices for this warp's NI fiber groups; the
// fragments of k-step kk + 1 are loaded (into the other register set) while k-step kk's DMMAs issue.
// Strips past the matrix (mi >= S1 / S2: zero rows of the padded factor) are read but skipped.
template <int MS, int NI, int NW, bool FWD, int KS, bool PS = false>
__device__ __forceinline__ void rchunk(const double* __restrict__ a1, const double* __restrict__ a2,
                                       const double* __restrict__ xa, const double* __restrict__ xb, int LDA,
                                       double (&c1)[MS][NI][2], double (&c2)[MS][NI][2]) {
    double av1[2][MS], av2[2][MS], b1[2][NI], b2[2][NI];
    rfrag<MS, NI, NW, FWD, PS>(a1, a2, xa, xb, LDA, 0, av1[0], av2[0], b1[0], b2[0]);
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
        const int cur = kk & 1, nxt = cur ^ 1;
        if (kk + 1 < KS) rfrag<MS, NI, NW, FWD, PS>(a1, a2, xa, xb, LDA, kk + 1, av1[nxt], av2[nxt], b1[nxt], b2[nxt]);
        // every strip unconditionally: padded strips are zero rows of the resident factors (a predicated
        // mma.sync costs a WARPSYNC + NOP per DMMA); their accumulators are never stored
#pragma unroll
        for (int mi = 0; mi < MS; ++mi) {
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) rdmma(c1[mi][ni][0], c1[mi][ni][1], av1[cur][mi], b1[cur][ni]);
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) rdmma(c2[mi][ni][0], c2[mi][ni][1], av2[cur][mi], b2[cur][ni]);
        }
    }
}

// Consumer warps: WS strip groups x WF fiber groups; warp (ws, wf) owns strips [ws MSW, ws MSW + MSW) of
// BOTH matrices and fiber groups [wf NI, wf NI + NI) of the tile.
template <int MS, int MSW, int NI, int WS, int WF, int NS, bool FWD, bool POST, bool PS = false>
__global__ void __launch_bounds__(32 * (WS * WF + 1), 1)
    fold_res_kernel(RArgs a, const double* __restrict__ X, double* __restrict__ Y, const double* __restrict__ J,
                    const double* __restrict__ post, const double* __restrict__ pre) {
    constexpr int NW = WS * WF;
    using SH = RShape<NI, WF, PS>;
    extern __shared__ __align__(16) double smem[];
    __shared__ uint64_t full[NS], empty[NS];
    const int LDA = a.LDA;
    constexpr int MR = 8 * MSW * WS;  // resident rows per matrix (strips past the factor: zero rows)
    double* sA = smem;                  // [2][MR][LDA]
    double* sX = smem + 2 * MR * LDA;   // [NS][STAGE]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

    // resident factors (both matrices), once per CTA
    for (int i = tid; i < 2 * MR * a.Kp; i += blockDim.x) {
        const int m = i / (MR * a.Kp), rem = i - m * MR * a.Kp;
        const int row = rem / a.Kp, col = rem - row * a.Kp;
        sA[(m * MR + row) * LDA + col] = row < a.Mp ? J[m * a.A2 + static_cast<long long>(row) * a.Kp + col] : 0.0;
    }
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
        // ---------------- producer warp ----------------
        // Address state per tile: L > 1: lane owns fibers lane + 32 u (pointer to row 0 of each);
        // L == 1: lane owns chunk row lane % 16 of fibers fp, fp + 2, ... (one pointer, step 2 n).
        // Interior chunks of full tiles take the unpredicated path (one 64-bit add per copy).
        unsigned seq = 0;
        for (long long tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
            const long long c0 = tile * SH::BN;
            const bool full_tile = c0 + SH::BN <= ncols;
            const double* fp0[SH::FPL];
            bool fv[SH::FPL];
            if (L != 1) {
#pragma unroll
                for (int u = 0; u < SH::FPL; ++u) {
                    const long long cc = c0 + lane + 32 * u;
                    fv[u] = cc < ncols && lane + 32 * u < SH::BN;
                    fp0[u] = X + rbase(fv[u] ? cc : 0, L, n);
                }
            }
            const int r16 = lane & 15, fpar = lane >> 4;
            const double* f1 = X + (full_tile || c0 + fpar < ncols ? c0 + fpar : 0) * n;
            if (POST) {  // the epilogue's D^-1/2 rows of this tile into L2, ~NQ chunks ahead of their use
                if (L != 1) {
#pragma unroll
                    for (int u = 0; u < SH::FPL; ++u)
                        if (fv[u] && (lane & 15) == 0)
                            for (int r = 0; r < n; ++r)
                                asm volatile("prefetch.global.L2 [%0];" ::"l"(post + (fp0[u] - X) + L * r));
                } else {
                    for (int f = lane; f < SH::BN; f += 32)
                        if (c0 + f < ncols)
                            for (int r = 0; r < n; r += 16)
                                asm volatile("prefetch.global.L2 [%0];" ::"l"(post + (c0 + f) * n + r));
                }
            }
            for (int q = 0; q < a.NQ; ++q, ++seq) {
                const int s = seq % NS;
                rmb_wait(&empty[s], ((seq / NS) & 1u) ^ 1u);
                const unsigned sa = ru32(sX + s * SH::STAGE), sb = sa + 8u * SH::XB;
                const unsigned dso = 8u * SH::DOFF;           // PS: D chunk bytes after its fiber chunk
                const long long dofs = PS ? pre - X : 0;      // D^-1/2 element = X element + dofs
                const int ra0 = q * kBK, rb0 = FWD ? n - q * kBK - kBK : a.F + q * kBK;
                const bool rows_in = ra0 + kBK <= n && rb0 >= 0 && rb0 + kBK <= n;
                if (L == 1) {
                    const int rowa = ra0 + r16, rowb = rb0 + r16;
                    const double* pa = f1 + rowa;
                    const double* pb = f1 + rowb;
                    const long long step = 2LL * n;
                    unsigned da = sa + 8u * (r16 * SH::LDX + fpar), db = sb + 8u * (r16 * SH::LDX + fpar);
                    if (full_tile && rows_in) {
#pragma unroll 8
                        for (int f = 0; f < SH::BN; f += 2) {
                            rcp8(da, pa, true);
                            rcp8(db, pb, true);
                            if (PS) {
                                rcp8(da + dso, pa + dofs, true);
                                rcp8(db + dso, pb + dofs, true);
                            }
                            pa += step;
                            pb += step;
                            da += 16u;
                            db += 16u;
                        }
                    } else {
                        const bool va = rowa < n, vb = rowb >= 0 && rowb < n;
                        for (int f = 0; f < SH::BN; f += 2) {
                            const bool cv = c0 + fpar + f < ncols;
                            rcp8(da, (va && cv) ? pa : X, va && cv);
                            rcp8(db, (vb && cv) ? pb : X, vb && cv);
                            if (PS) {
                                rcp8(da + dso, (va && cv) ? pa + dofs : X, va && cv);
                                rcp8(db + dso, (vb && cv) ? pb + dofs : X, vb && cv);
                            }
                            pa += step;
                            pb += step;
                            da += 16u;
                            db += 16u;
                        }
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < SH::FPL; ++u) {
                        if (SH::BN % 32 != 0 && lane + 32 * u >= SH::BN) continue;
                        const double* pa = fp0[u] + L * ra0;
                        const double* pb = fp0[u] + L * rb0;
                        unsigned da = sa + 8u * (lane + 32 * u), db = sb + 8u * (lane + 32 * u);
                        if (fv[u] && rows_in) {
#pragma unroll 8
                            for (int r = 0; r < kBK; ++r) {
                                rcp8(da, pa, true);
                                rcp8(db, pb, true);
                                if (PS) {
                                    rcp8(da + dso, pa + dofs, true);
                                    rcp8(db + dso, pb + dofs, true);
                                }
                                pa += L;
                                pb += L;
                                da += 8u * SH::LDX;
                                db += 8u * SH::LDX;
                            }
                        } else {
                            for (int r = 0; r < kBK; ++r) {
                                const bool va = fv[u] && ra0 + r < n, vb = fv[u] && rb0 + r >= 0 && rb0 + r < n;
                                rcp8(da, va ? pa : X, va);
                                rcp8(db, vb ? pb : X, vb);
                                if (PS) {
                                    rcp8(da + dso, va ? pa + dofs : X, va);
                                    rcp8(db + dso, vb ? pb + dofs : X, vb);
                                }
                                pa += L;
                                pb += L;
                                da += 8u * SH::LDX;
                                db += 8u * SH::LDX;
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
    const int so = ws * MSW;  // first strip of this warp
    const double* a1 = sA + (so * 8 + g) * LDA + t;
    const double* a2 = sA + MR * LDA + (so * 8 + g) * LDA + t;
    const int fcol = wf * NI * 8 + g;  // this lane's B-fragment fiber column within the tile
    unsigned seq = 0;
    for (long long tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
        const long long c0 = tile * SH::BN;
        double c1[MSW][NI][2], c2[MSW][NI][2];
#pragma unroll
        for (int mi = 0; mi < MSW; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) c1[mi][ni][0] = c1[mi][ni][1] = c2[mi][ni][0] = c2[mi][ni][1] = 0.0;
        for (int q = 0; q < a.NQ; ++q, ++seq) {
            const int s = seq % NS;
            rmb_wait(&full[s], (seq / NS) & 1u);
            const double* st = sX + s * SH::STAGE;
            const double* xa = st + t * SH::LDX + fcol;
            const double* xb = st + SH::XB + (FWD ? (kBK - 1 - t) : t) * SH::LDX + fcol;
            const int k0 = q * kBK;
            const int ks = min(kBK, a.Kp - k0) >> 2;
            if (ks == 4) rchunk<MSW, NI, WF, FWD, 4, PS>(a1 + k0, a2 + k0, xa, xb, LDA, c1, c2);
            else if (ks == 3) rchunk<MSW, NI, WF, FWD, 3, PS>(a1 + k0, a2 + k0, xa, xb, LDA, c1, c2);
            else if (ks == 2) rchunk<MSW, NI, WF, FWD, 2, PS>(a1 + k0, a2 + k0, xa, xb, LDA, c1, c2);
            else rchunk<MSW, NI, WF, FWD, 1, PS>(a1 + k0, a2 + k0, xa, xb, LDA, c1, c2);
            __syncwarp();
            if (lane == 0) rmb_arrive(&empty[s]);
        }
        // register epilogue (same output mapping as fold_mode_kernel)
        long long ob[NI][2];
        bool cv[NI][2];
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const long long cc = c0 + (wf * NI + ni) * 8 + 2 * t + v;
                cv[ni][v] = cc < ncols;
                ob[ni][v] = rbase(cv[ni][v] ? cc : 0, L, n);
            }
        if constexpr (POST) {
            // D^-1/2 post-scale: every scale value of the tile is loaded (into the dead fragment
            // registers) before the first store; the producer prefetched these rows into L2
            double pl[MSW][NI][2], ph[MSW][NI][2];
#pragma unroll
            for (int mi = 0; mi < MSW; ++mi) {
                const int i = (so + mi) * 8 + g;
                const int ilo = i < a.F ? i : 0, ihi = i < a.h ? n - 1 - i : 0;
#pragma unroll
                for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                    for (int v = 0; v < 2; ++v) {
                        pl[mi][ni][v] = cv[ni][v] ? __ldg(post + ob[ni][v] + L * ilo) : 0.0;
                        ph[mi][ni][v] = cv[ni][v] ? __ldg(post + ob[ni][v] + L * ihi) : 0.0;
                    }
            }
#pragma unroll
            for (int mi = 0; mi < MSW; ++mi) {
                const int i = (so + mi) * 8 + g;
#pragma unroll
                for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                    for (int v = 0; v < 2; ++v) {
                        if (!cv[ni][v]) continue;
                        double* y = Y + ob[ni][v];
                        if (i < a.h) {
                            y[L * i] = pl[mi][ni][v] * (c1[mi][ni][v] + c2[mi][ni][v]);
                            y[L * (n - 1 - i)] = ph[mi][ni][v] * (c1[mi][ni][v] - c2[mi][ni][v]);
                        } else if (i < a.F) {  // middle row (odd n)
                            y[L * i] = pl[mi][ni][v] * c1[mi][ni][v];
                        }
                    }
            }
            continue;
        }
#pragma unroll
        for (int mi = 0; mi < MSW; ++mi) {
            const int i = (so + mi) * 8 + g;
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    if (!cv[ni][v]) continue;
                    double* y = Y + ob[ni][v];
                    if (FWD) {
                        if (i < a.F) y[L * i] = c1[mi][ni][v];
                        if (i < a.h) y[L * (a.F + i)] = c2[mi][ni][v];
                    } else if (i < a.h) {
                        double lo = c1[mi][ni][v] + c2[mi][ni][v], hi = c1[mi][ni][v] - c2[mi][ni][v];
                        if (POST) {
                            lo *= __ldg(post + ob[ni][v] + L * i);
                            hi *= __ldg(post + ob[ni][v] + L * (n - 1 - i));
                        }
                        y[L * i] = lo;
                        y[L * (n - 1 - i)] = hi;
                    } else if (i < a.F) {  // middle row (odd n)
                        double mid = c1[mi][ni][v];
                        if (POST) mid *= __ldg(post + ob[ni][v] + L * i);
                        y[L * i] = mid;
                    }
                }
        }
    }
}

int lda_of(int Kp) { return Kp + ((4 - Kp % 16) % 16 + 16) % 16; }

size_t res_smem(int MSWS, int NI, int WF, int NS, int Kp, bool ps = false) {  // MSWS = strips per warp x groups
    const int BN = 8 * NI * WF;
    return sizeof(double) *
           (2 * 8 * static_cast<size_t>(MSWS) * lda_of(Kp) + static_cast<size_t>(NS) * 2 * kBK * (BN + 4) * (ps ? 2 : 1));
}

RArgs make_rargs(const Tiling& t, const ModeGeom& g) {
    RArgs a;
    a.geo = g;
    a.h = g.n / 2;
    a.F = g.n - a.h;
    a.Kp = t.Kp;
    a.LDA = lda_of(t.Kp);
    a.NQ = (t.Kp + kBK - 1) / kBK;
    a.S1 = (a.F + 7) / 8;
    a.S2 = (a.h + 7) / 8;
    a.A2 = static_cast<long long>(t.Mp) * t.Kp;
    a.Mp = t.Mp;
    a.ntiles = (g.ncols + t.BN - 1) / t.BN;
    return a;
}

int g_sms = 0;

template <int MS, int MSW, int NI, int WS, int WF, int NS>
cudaError_t res_launch_t(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J, bool fwd,
                         const double* post, const double* pre, cudaStream_t st, int* occ) {
    constexpr int NW = WS * WF;
    auto k = fwd ? (pre ? fold_res_kernel<MS, MSW, NI, WS, WF, NS, true, false, true>
                        : fold_res_kernel<MS, MSW, NI, WS, WF, NS, true, false>)
                 : (post ? fold_res_kernel<MS, MSW, NI, WS, WF, NS, false, true>
                         : fold_res_kernel<MS, MSW, NI, WS, WF, NS, false, false>);
    const size_t smem = res_smem(MSW * WS, NI, WF, NS, t.Kp, pre != nullptr);
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
    if (g_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_sms <= 0) g_sms = 148;
    }
    const RArgs ra = make_rargs(t, g);
    const long long grid = std::min<long long>(ra.ntiles, static_cast<long long>(g_sms) * std::max(1, t.ctas_per_sm));
    k<<<static_cast<unsigned>(grid), 32 * (NW + 1), smem, st>>>(ra, X, Y, J, post, pre);
    return cudaGetLastError();
}

template <int MS>
cudaError_t res_dispatch_ms(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J, bool fwd,
                            const double* post, const double* pre, cudaStream_t st, int* occ) {
    // (NI, NW, NS) variants
    // Tiling fields: WM = strip groups (WS), WN = fiber groups (WF), NI, nstage.  Consumer warps + 1
    // producer stay <= 8 warps (a 9-warp CTA caps the registers at 168).
    constexpr int H = (MS + 1) / 2;  // strips per warp with two strip groups
    if (t.WM == 1 && t.NI == 1 && t.WN == 7 && t.nstage == 4) return res_launch_t<MS, MS, 1, 1, 7, 4>(t, g, X, Y, J, fwd, post, pre, st, occ);
    // 8 consumer warps = two per SM sub-partition (a warp issues at most one DMMA.8x8x4 per 16 cycles,
    // the sub-partition's DMMA unit accepts one per ~16: two ready warps per sub-partition keep it fed)
    if (t.WM == 1 && t.NI == 1 && t.WN == 8 && t.nstage == 4) return res_launch_t<MS, MS, 1, 1, 8, 4>(t, g, X, Y, J, fwd, post, pre, st, occ);
    if (t.WM == 1 && t.NI == 1 && t.WN == 8 && t.nstage == 2) return res_launch_t<MS, MS, 1, 1, 8, 2>(t, g, X, Y, J, fwd, post, pre, st, occ);
    if (t.WM == 2 && t.NI == 1 && t.WN == 4 && t.nstage == 4) return res_launch_t<MS, H, 1, 2, 4, 4>(t, g, X, Y, J, fwd, post, pre, st, occ);
    // 12 consumer warps (three per sub-partition), half the strips each
    if (t.WM == 2 && t.NI == 1 && t.WN == 6 && t.nstage == 4) return res_launch_t<MS, H, 1, 2, 6, 4>(t, g, X, Y, J, fwd, post, pre, st, occ);
    if (t.WM == 2 && t.NI == 1 && t.WN == 6 && t.nstage == 2) return res_launch_t<MS, H, 1, 2, 6, 2>(t, g, X, Y, J, fwd, post, pre, st, occ);
    if (t.WM == 2 && t.NI == 2 && t.WN == 3 && t.nstage == 4) return res_launch_t<MS, H, 2, 2, 3, 4>(t, g, X, Y, J, fwd, post, pre, st, occ);
    if (t.WM == 2 && t.NI == 1 && t.WN == 3 && t.nstage == 6) return res_launch_t<MS, H, 1, 2, 3, 6>(t, g, X, Y, J, fwd, post, pre, st, occ);
    if constexpr (MS <= 8) {
        if (t.WM == 1 && t.NI == 2 && t.WN == 4 && t.nstage == 4) return res_launch_t<MS, MS, 2, 1, 4, 4>(t, g, X, Y, J, fwd, post, pre, st, occ);
    }
    return cudaErrorInvalidValue;
}

cudaError_t res_dispatch(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* J, bool fwd,
                         const double* post, const double* pre, cudaStream_t st, int* occ) {
    switch (t.MI) {
        case 4: return res_dispatch_ms<4>(t, g, X, Y, J, fwd, post, pre, st, occ);
        case 5: return res_dispatch_ms<5>(t, g, X, Y, J, fwd, post, pre, st, occ);
        case 6: return res_dispatch_ms<6>(t, g, X, Y, J, fwd, post, pre, st, occ);
        case 7: return res_dispatch_ms<7>(t, g, X, Y, J, fwd, post, pre, st, occ);
        case 8: return res_dispatch_ms<8>(t, g, X, Y, J, fwd, post, pre, st, occ);
        case 9: return res_dispatch_ms<9>(t, g, X, Y, J, fwd, post, pre, st, occ);
        case 10: return res_dispatch_ms<10>(t, g, X, Y, J, fwd, post, pre, st, occ);
        case 11: return res_dispatch_ms<11>(t, g, X, Y, J, fwd, post, pre, st, occ);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

std::vector<Tiling> fold_res_candidates(int n, int Mp_hint) {
    std::vector<Tiling> out;
    const int h = n / 2, F = n - h;
    if (h < 1) return out;
    const int S = (F + 7) / 8;
    if (S < 4 || S > 11) return out;  // small factors: the streaming kernel; n > 176: factors exceed smem
    const int Kp = (F + 3) / 4 * 4;
    // WM(WS), NI, WN(WF), NS; {1, 1, 8, 2}: the fused D^-1/2 pre-scale variant (doubled stages fit)
    const int variants[8][4] = {{1, 1, 8, 4}, {2, 1, 4, 4}, {1, 1, 7, 4}, {2, 2, 3, 4}, {1, 2, 4, 4}, {1, 1, 8, 2},
                                {2, 1, 6, 4}, {2, 1, 6, 2}};
    for (const auto& v : variants) {
        Tiling t;
        t.fold = 2;
        t.MI = S;
        t.WM = v[0];
        t.NI = v[1];
        t.WN = v[2];
        t.nstage = v[3];
        t.S = S;
        t.RB = 1;
        t.MpB = 8 * S;
        t.Mp = std::max(8 * S, Mp_hint);
        t.Kp = Kp;
        t.BN = 8 * t.NI * t.WN;
        t.LDX = t.BN + 4;
        t.smem = res_smem(t.WM == 2 ? 2 * ((S + 1) / 2) : S, t.NI, t.WN, t.nstage, Kp);
        if (t.smem + 1024 > kSmemPerCTA) continue;
        if (t.WM == 1 && t.NI == 2 && S > 8) continue;  // 4 S NI accumulator doubles: spills beyond S = 8
        int occ = 0;
        res_dispatch(t, ModeGeom{}, nullptr, nullptr, nullptr, true, nullptr, nullptr, nullptr, &occ);
        if (occ < 1) continue;
        t.ctas_per_sm = 1;
        out.push_back(t);
    }
    return out;
}

cudaError_t launch_fold_res(const Tiling& t, const ModeGeom& g, const double* X, double* Y, const double* Jfold,
                            bool forward, const double* post_scale, cudaStream_t st, const double* pre_scale) {
    if (g.ncols <= 0) return cudaSuccess;
    if (t.fold != 2 || g.m != g.n || g.n < 2 || (forward && post_scale) || (!forward && pre_scale))
        return cudaErrorInvalidValue;
    if (pre_scale && fold_res_prescale_smem(t) + 1024 > kSmemPerCTA) return cudaErrorInvalidValue;
    return res_dispatch(t, g, X, Y, Jfold, forward, post_scale, pre_scale, st, nullptr);
}

size_t fold_res_prescale_smem(const Tiling& t) {
    return res_smem(t.WM == 2 ? 2 * ((t.MI + 1) / 2) : t.MI, t.NI, t.WN, t.nstage, t.Kp, true);
}

}  // namespace gpu
}  // namespace stiga
