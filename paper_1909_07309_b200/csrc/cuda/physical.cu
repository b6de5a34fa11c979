// Physical spatial stiffness / mass assembly (one CTA per element, geometry evaluated in-kernel)
// and the stencil SpMM of the space-time system mat-vec.  See physical.cuh.
#include "physical.cuh"
#include "geom_device.cuh"

#include <cuda.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

namespace stiga {
namespace gpu {

namespace {

using namespace geomdev;

// One CTA per element: quadrature-point geometry factors G = w det nu J^-1 J^-T and w det gamma in
// smem, then every (a, b) pair of local functions, atomically added into the stencil rows.
template <int D>
__global__ void __launch_bounds__(256) physical_assembly_kernel(PhysicalDesc g, double* Kst, double* Mst) {
    constexpr int NG = D * (D + 1) / 2 + 1;  // unique G entries + mass weight
    extern __shared__ double sm[];
    const int q = g.q, P1 = g.p + 1;
    int QD = 1, LD = 1;
    for (int l = 0; l < D; ++l) {
        QD *= q;
        LD *= P1;
    }
    double* gq = sm;                     // QD x NG
    double* tv = gq + QD * NG;           // D x q x P1 values
    double* td = tv + D * q * P1;        // D x q x P1 derivatives
    int* firstl = reinterpret_cast<int*>(td + D * q * P1);  // D
    int e[D];
    {
        long long rem = blockIdx.x;
        for (int l = 0; l < D; ++l) {
            e[l] = static_cast<int>(rem % g.n_el);
            rem /= g.n_el;
        }
    }
    for (int i = threadIdx.x; i < D * q * P1; i += blockDim.x) {
        const int l = i / (q * P1), r = i % (q * P1);
        const int src = (e[l] * q) * P1 + r;
        tv[i] = g.bval[src];
        td[i] = g.bder[src];
    }
    if (threadIdx.x < D) firstl[threadIdx.x] = g.bfirst[e[threadIdx.x] * q];
    for (int qi = threadIdx.x; qi < QD; qi += blockDim.x) {
        double eta[D], w = 1.0;
        int rem = qi;
        for (int l = 0; l < D; ++l) {
            const int jl = rem % q;
            rem /= q;
            eta[l] = g.qnode[e[l] * q + jl];
            w *= g.qweight[e[l] * q + jl];
        }
        double x[D], J[D * D], Ji[D * D];
        geometry_eval<D>(g, eta, x, J);
        const double det = det_inv<D>(J, Ji);
        const double nu = field(g.nu_kind, x), gam = field(g.gamma_kind, x);
        int k = 0;
        for (int r = 0; r < D; ++r)
            for (int c = r; c < D; ++c) {
                double s = 0.0;  // (J^-1 J^-T)_{rc} = sum_m Ji[r][m] Ji[c][m]
                for (int m = 0; m < D; ++m) s += Ji[r + D * m] * Ji[c + D * m];
                gq[qi * NG + k++] = w * det * nu * s;
            }
        gq[qi * NG + NG - 1] = w * det * gam;
    }
    __syncthreads();
    const int W = 2 * g.p + 1;
    long long ostride[D], nstride[D];
    {
        long long o = 1, s = 1;
        for (int l = 0; l < D; ++l) {
            ostride[l] = o;
            nstride[l] = s;
            o *= W;
            s *= g.n;
        }
    }
    const long long Ns = nstride[D - 1] * g.n;
    for (int pair = threadIdx.x; pair < LD * LD; pair += blockDim.x) {
        const int ia = pair % LD, ib = pair / LD;
        int a[D], b[D], ga[D], gb[D];
        bool ok = true;
        {
            int ra = ia, rb = ib;
            for (int l = 0; l < D; ++l) {
                a[l] = ra % P1;
                ra /= P1;
                b[l] = rb % P1;
                rb /= P1;
                ga[l] = firstl[l] + a[l];
                gb[l] = firstl[l] + b[l];
                ok = ok && ga[l] >= 0 && ga[l] < g.n && gb[l] >= 0 && gb[l] < g.n;
            }
        }
        if (!ok) continue;
        double kab = 0.0, mab = 0.0;
        for (int qi = 0; qi < QD; ++qi) {
            int j[D];
            int rem = qi;
            for (int l = 0; l < D; ++l) {
                j[l] = rem % q;
                rem /= q;
            }
            double va = 1.0, vb = 1.0, da[D], db[D];
            for (int c = 0; c < D; ++c) da[c] = db[c] = 1.0;
            for (int l = 0; l < D; ++l) {
                const double vla = tv[(l * q + j[l]) * P1 + a[l]], dla = td[(l * q + j[l]) * P1 + a[l]];
                const double vlb = tv[(l * q + j[l]) * P1 + b[l]], dlb = td[(l * q + j[l]) * P1 + b[l]];
                va *= vla;
                vb *= vlb;
                for (int c = 0; c < D; ++c) {
                    da[c] *= (c == l) ? dla : vla;
                    db[c] *= (c == l) ? dlb : vlb;
                }
            }
            const double* G = gq + qi * NG;
            double s = 0.0;
            int k = 0;
            for (int r = 0; r < D; ++r)
                for (int c = r; c < D; ++c) {
                    const double gv = G[k++];
                    s += (r == c) ? gv * da[r] * db[r] : gv * (da[r] * db[c] + da[c] * db[r]);
                }
            kab += s;
            mab += G[NG - 1] * va * vb;
        }
        long long row = 0, off = 0;
        for (int l = 0; l < D; ++l) {
            row += ga[l] * nstride[l];
            off += (gb[l] - ga[l] + g.p) * ostride[l];
        }
        atomicAdd(Kst + off * Ns + row, kab);  // offset-major: rows of one offset contiguous
        atomicAdd(Mst + off * Ns + row, mab);
    }
}

// MX = M_s X and KX = K_s X for X (N_s x n_t, colex) on the FP64 tensor cores (DMMA m8n8k4).
//
// The stencil rows of 8 consecutive i_1 (fixed i_2.., one neighbour-line offset (o_2, o_3)) touch the
// window of 8 + 2p neighbours j_1 = i_1 - p .. i_1 + 7 + p, so for that offset the contribution is a
// dense 8 x 4KS block (the band, zero outside |j_1 - i_1| <= p) times the window of the neighbour
// line: y[8 rows, t] += A_band (8 x 4KS) * X[window, t].  One CTA owns a segment of up to 8*NW rows
// of one line (consumer warp w = rows 8w..8w+7) and the t of its chunk, and walks the (2p+1)^(d-1)
// neighbour lines: each step stages one neighbour-line segment (+-p halo) x t-chunk [t][row] (row
// pitch == 4 mod 16 doubles: conflict-free B fragments) and the segment's band values [o_1][row].
// M and K share the staged X, so each B fragment feeds two DMMAs.
//
// Two stagings: (a) n even (TMA-legal strides): one producer lane issues three TMA tensor loads
// per step (X box, M and K band boxes; out-of-range rows / t zero-filled by the TMA unit) into a
// kStages ring guarded by full / empty mbarriers, consumers never meet a CTA barrier;
// (b) otherwise every thread stages with 8-byte cp.async (double buffered, one CTA barrier a step).
// A third kernel, (c) further down, takes the 8 MMA rows from two neighbouring lines (line-pair bricks:
// denser band blocks); it is the one selected for d >= 2, n even, n <= 72 (BASELINE configs[3]).
constexpr int kTT = 9;          // 8-column time tiles per chunk (72 columns)
constexpr int kMaxWarps = 12;   // row blocks per CTA (96 rows); two consumer warps (M, K) each
constexpr int kStages = 3;

__device__ __forceinline__ void sdmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ void scp8(unsigned dst, const double* src, bool valid) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ unsigned su32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mb_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count));
}
__device__ __forceinline__ void mb_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void mb_expect(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(su32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma3(unsigned dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(su32(bar))
        : "memory");
}
__device__ __forceinline__ void tma2(unsigned dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(su32(bar))
        : "memory");
}

struct StencilGeo {
    int n, p, W, d;
    long long Ns;
    int n_t;
    int nseg, seg_rows;  // segments per line, rows per segment (multiple of 8)
    int SR, LDR;         // staged rows per neighbour line and their smem pitch (== 4 mod 16)
    int BR;              // band smem pitch (rows) == seg_rows
    int nsteps;          // W^(d-1) neighbour-line offsets
    int xstage, bstage;  // doubles per X / band stage (multiples of 16: 128-byte aligned stages)
    int shift;           // staged window starts at row seg0 - p - shift (TMA: even start coordinate)
    int nst;             // TMA ring depth
    int boxt;            // time columns per TMA box (min(72, n_t))
};

struct LineCtx {
    int lc[2];
    long long line;
    int seg0, t0, tcols;
};

__device__ __forceinline__ LineCtx line_ctx(const StencilGeo& sg) {
    LineCtx c;
    c.line = blockIdx.x / sg.nseg;  // i_2 + n i_3 (0 for d = 1)
    c.seg0 = static_cast<int>(blockIdx.x % sg.nseg) * sg.seg_rows;
    c.t0 = blockIdx.y * (8 * kTT);
    c.tcols = min(8 * kTT, sg.n_t - c.t0);
    c.lc[0] = c.lc[1] = 0;
    long long r = c.line;
    for (int l = 0; l < sg.d - 1; ++l) {
        c.lc[l] = static_cast<int>(r % sg.n);
        r /= sg.n;
    }
    return c;
}

// The valid steps of a line are the rectangle of neighbour offsets inside the patch; StepIter walks it with
// counters (nb_line / next_step cost an integer division per step and warp, ~15% of the issue slots of the
// line-pair kernel before it switched to counters).
struct StepIter {
    int o2, o3, lo2, hi2, hi3;
    long long base;  // neighbour line of (o2, o3) = base + o2 + n o3
    int n, W;
    __device__ __forceinline__ StepIter(const StencilGeo& sg, const LineCtx& c) : n(sg.n), W(sg.W) {
        if (sg.d == 1) {
            lo2 = hi2 = 0;
            o3 = hi3 = 0;
            base = 0;
        } else {
            lo2 = max(0, sg.p - c.lc[0]);
            hi2 = min(sg.W - 1, sg.n - 1 - c.lc[0] + sg.p);
            const int lo3 = sg.d < 3 ? 0 : max(0, sg.p - c.lc[1]);
            hi3 = sg.d < 3 ? 0 : min(sg.W - 1, sg.n - 1 - c.lc[1] + sg.p);
            o3 = lo3;
            base = (c.lc[0] - sg.p) + (sg.d < 3 ? 0LL : static_cast<long long>(sg.n) * (c.lc[1] - sg.p));
        }
        o2 = lo2;
    }
    __device__ __forceinline__ bool valid() const { return o3 <= hi3; }
    __device__ __forceinline__ int step() const { return o2 + W * o3; }  // offset-plane group index
    __device__ __forceinline__ long long line() const { return base + o2 + static_cast<long long>(n) * o3; }
    __device__ __forceinline__ void next() {
        if (++o2 > hi2) {
            o2 = lo2;
            ++o3;
        }
    }
};

// One step of a consumer warp: accumulate the band of offset step into (accm, acck).
// One step of consumer warp (row block rb, matrix mat): acc += band(mat) x staged window.
template <int KS, bool FULL>
__device__ __forceinline__ void stencil_step_t(const StencilGeo& sg, const double* xs, const double* bm, int rb,
                                               int ntiles, double (&acc)[kTT][2]) {
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2, t4 = lane & 3;
    const double* bs = xs + g * sg.LDR + sg.shift + 8 * rb + t4;
    const double* br = bm + 8 * rb + g;
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
        const int o1 = 4 * kk + t4 - g;
        const bool av = o1 >= 0 && o1 < sg.W;
        const double a = av ? br[av ? o1 * sg.BR : 0] : 0.0;  // clamped index: the load is unconditional
#pragma unroll
        for (int tt = 0; tt < kTT; ++tt) {
            if (FULL || tt < ntiles) sdmma(acc[tt][0], acc[tt][1], a, bs[tt * 8 * sg.LDR + 4 * kk]);
        }
    }
}

template <int KS>
__device__ __forceinline__ void stencil_step(const StencilGeo& sg, const double* xs, const double* bm, int rb,
                                             int ntiles, double (&acc)[kTT][2]) {
    if (ntiles == kTT) stencil_step_t<KS, true>(sg, xs, bm, rb, ntiles, acc);
    else stencil_step_t<KS, false>(sg, xs, bm, rb, ntiles, acc);
}

__device__ __forceinline__ void stencil_store(const StencilGeo& sg, const LineCtx& c, int rb,
                                              const double (&acc)[kTT][2], double* Y) {
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2, t4 = lane & 3;
    const int i1 = c.seg0 + 8 * rb + g;
    if (i1 >= sg.n) return;
    const long long irow = i1 + sg.n * c.line;
    // C fragment: row g, columns 2 t4 + {0, 1} of tile tt
#pragma unroll
    for (int tt = 0; tt < kTT; ++tt) {
#pragma unroll
        for (int v = 0; v < 2; ++v) {
            const int tc = 8 * tt + 2 * t4 + v;
            if (tc < c.tcols) Y[irow + sg.Ns * (c.t0 + tc)] = acc[tt][v];
        }
    }
}

// (a) TMA staging, warp-specialized: warps 0..nwc-1 consume (row block w % nrb, matrix w / nrb),
// warp nwc produces.
template <int KS>
__global__ void __launch_bounds__(32 * (2 * kMaxWarps + 1))
    stencil_tma_kernel(StencilGeo sg, const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapM,
                       const __grid_constant__ CUtensorMap mapK, double* __restrict__ MX, double* __restrict__ KX) {
    extern __shared__ __align__(128) double sx[];
    const int nst = sg.nst;
    double* xs = sx;                     // nst x xstage
    double* bsm = xs + nst * sg.xstage;  // nst x (M, K) x bstage
    uint64_t* full = reinterpret_cast<uint64_t*>(bsm + nst * 2 * sg.bstage);
    uint64_t* empty = full + nst;
    const int nwc = blockDim.x / 32 - 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const LineCtx c = line_ctx(sg);
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            mb_init(full + s, 1);
            mb_init(empty + s, nwc);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (warp == nwc) {
        if (lane != 0) return;
        const unsigned bytes = 8u * (sg.boxt * sg.LDR + 2 * sg.W * sg.BR);
        const int row0 = static_cast<int>(c.seg0 + sg.n * c.line);
        int k = 0;
        for (StepIter it(sg, c); it.valid(); it.next(), ++k) {
            const int st = k % nst;
            if (k >= nst) mb_wait(empty + st, ((k / nst) - 1) & 1);
            mb_expect(full + st, bytes);
            tma3(su32(xs + st * sg.xstage), &mapX, c.seg0 - sg.p - sg.shift, static_cast<int>(it.line()), c.t0, full + st);
            tma2(su32(bsm + (st * 2) * sg.bstage), &mapM, row0, sg.W * it.step(), full + st);
            tma2(su32(bsm + (st * 2 + 1) * sg.bstage), &mapK, row0, sg.W * it.step(), full + st);
        }
        return;
    }
    const int nrb = nwc / 2, rb = warp % nrb, mat = warp / nrb;
    const int ntiles = (c.tcols + 7) >> 3;
    double acc[kTT][2];
#pragma unroll
    for (int t = 0; t < kTT; ++t) acc[t][0] = acc[t][1] = 0.0;
    int k = 0;
    for (StepIter it(sg, c); it.valid(); it.next(), ++k) {
        const int st = k % nst;
        mb_wait(full + st, (k / nst) & 1);
        stencil_step<KS>(sg, xs + st * sg.xstage, bsm + (st * 2 + mat) * sg.bstage, rb, ntiles, acc);
        __syncwarp();
        if (lane == 0) mb_arrive(empty + st);
    }
    stencil_store(sg, c, rb, acc, mat ? KX : MX);
}

// (c) Line-pair bricks (n even, <= 72 rows per line, d >= 2): the 8 MMA rows are 4 consecutive i_1 of
// TWO neighbouring lines (i_2 = 2q, 2q + 1) instead of 8 consecutive i_1 of one line.  The union of the
// 8 rows' neighbour windows is (4 + 2p) x (2p + 2) lines instead of (8 + 2p) x (2p + 1): for p = 4 the
// band blocks are 9/12 * 9/10 = 67% dense instead of 9/16 = 56%, and 66 rows pad to 68 instead of 72 --
// 17% fewer DMMAs per output row.  A CTA owns a line pair and <= 72 time columns and walks the
// (2p + 2) * (2p + 1)^(d-2) neighbour lines j_2 = 2q - p + e; at step e line a uses offset plane o_2 = e - p
// (e <= 2p), line b plane o_2 = e - p - 1 (e >= 1); the missing band of the first / last step is a zero
// A-fragment half (warp-uniform flag).  Consumer warp = 3 row blocks x one matrix; same TMA ring.
struct PairGeo {
    int n, p, W, d;
    long long Ns;
    int n_t;
    int nblk;            // 4-row blocks per line
    int LDR, BR;         // X-window / band smem pitches (== 4 mod 16)
    int nsteps;          // (W + 1) * W^(d-2)
    int xstage, bstage;  // doubles per X stage / per (matrix, line) band stage
    int shift, nst, boxt;
};

struct PairCtx {
    int i2, i3, t0, tcols;
    long long line_a;
};

__device__ __forceinline__ PairCtx pair_ctx(const PairGeo& sg) {
    PairCtx c;
    const int half = sg.n / 2;
    c.i2 = 2 * static_cast<int>(blockIdx.x % half);
    c.i3 = static_cast<int>(blockIdx.x / half);  // 0 for d = 2
    c.line_a = c.i2 + static_cast<long long>(sg.n) * c.i3;
    c.t0 = blockIdx.y * (8 * kTT);
    c.tcols = min(8 * kTT, sg.n_t - c.t0);
    return c;
}

template <int KS, bool FULL>
__device__ __forceinline__ void pair_step_t(const PairGeo& sg, const double* xs, const double* bm, int rb, bool va,
                                            bool vb, int ntiles, double (&acc)[kTT][2]) {
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2, t4 = lane & 3;
    const int ln = g >> 2, gi = g & 3;
    const bool lv = ln ? vb : va;
    const double* bs = xs + g * sg.LDR + sg.shift + 4 * rb + t4;
    const double* br = bm + ln * sg.bstage + 4 * rb + gi;
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
        const int o1 = 4 * kk + t4 - gi;
        const bool av = lv && o1 >= 0 && o1 < sg.W;
        const double a = av ? br[av ? o1 * sg.BR : 0] : 0.0;
#pragma unroll
        for (int tt = 0; tt < kTT; ++tt) {
            if (FULL || tt < ntiles) sdmma(acc[tt][0], acc[tt][1], a, bs[tt * 8 * sg.LDR + 4 * kk]);
        }
    }
}

// All RBW consecutive row blocks of a warp in one pass: row block r and contraction chunk kk read window
// columns 4 (rb0 + r + kk) .., so the RBW * KS (block, chunk) pairs share RBW + KS - 1 distinct B fragments
// per time tile (5 instead of 9 loads for RBW = KS = 3).  Per accumulator the chunks are still added in
// ascending kk, i.e. the same order as pair_step_t.  NR = live row blocks (RBW, or fewer for the last warp).
template <int KS, int RBW, int NR, bool FULL>
__device__ __forceinline__ void pair_step_all(const PairGeo& sg, const double* xs, const double* bm, int rb0, bool va,
                                              bool vb, int ntiles, double (&acc)[RBW][kTT][2]) {
    const int lane = threadIdx.x & 31;
    const int g = lane >> 2, t4 = lane & 3;
    const int ln = g >> 2, gi = g & 3;
    const bool lv = ln ? vb : va;
    const double* bs = xs + g * sg.LDR + sg.shift + 4 * rb0 + t4;
    const double* br = bm + ln * sg.bstage + 4 * rb0 + gi;
    double a[NR][KS];
#pragma unroll
    for (int kk = 0; kk < KS; ++kk) {
        const int o1 = 4 * kk + t4 - gi;
        const bool av = lv && o1 >= 0 && o1 < sg.W;
        const int off = av ? o1 * sg.BR : 0;
#pragma unroll
        for (int r = 0; r < NR; ++r) a[r][kk] = av ? br[off + 4 * r] : 0.0;
    }
#pragma unroll
    for (int tt = 0; tt < kTT; ++tt) {
        if (FULL || tt < ntiles) {
#pragma unroll
            for (int cc = 0; cc < NR + KS - 1; ++cc) {
                const double b = bs[tt * 8 * sg.LDR + 4 * cc];
#pragma unroll
                for (int r = 0; r < NR; ++r) {
                    const int kk = cc - r;
                    if (kk >= 0 && kk < KS) sdmma(acc[r][tt][0], acc[r][tt][1], a[r][kk], b);
                }
            }
        }
    }
}

// Registers are allocated to warps in groups of four, so a 13th (producer) warp would cap the kernel at 128
// registers and spill the 3 x 9 accumulator tiles: the producer is lane 0 of consumer warp 0 instead (it
// issues the loads of step k + nst - 1 before computing step k), 12 warps, <= 168 registers.
template <int KS, int RBW>
__global__ void __launch_bounds__(32 * 2 * ((18 + RBW - 1) / RBW))
    stencil_pair_kernel(PairGeo sg, const __grid_constant__ CUtensorMap mapX, const __grid_constant__ CUtensorMap mapM,
                        const __grid_constant__ CUtensorMap mapK, double* __restrict__ MX, double* __restrict__ KX) {
    extern __shared__ __align__(128) double sx[];
    const int nst = sg.nst;
    double* xs = sx;                     // nst x xstage
    double* bsm = xs + nst * sg.xstage;  // nst x (M, K) x (line a, line b) x bstage
    uint64_t* full = reinterpret_cast<uint64_t*>(bsm + nst * 4 * sg.bstage);
    uint64_t* empty = full + nst;
    const int nwc = blockDim.x / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const PairCtx c = pair_ctx(sg);
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            mb_init(full + s, 1);
            mb_init(empty + s, nwc);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    // Valid steps = the rectangle of neighbour offsets inside the patch: e in [e_lo, e_hi] (j_2 = i_2 - p + e),
    // o_3 in [o_lo, o_hi] (j_3 = i_3 - p + o_3); walked with incremental counters (an integer division per
    // step and warp showed up as ~15% of the issue slots in the first version).
    const int e_lo = max(0, sg.p - c.i2), e_hi = min(sg.W, sg.n - 1 - c.i2 + sg.p);
    const int o_lo = sg.d < 3 ? 0 : max(0, sg.p - c.i3), o_hi = sg.d < 3 ? 0 : min(sg.W - 1, sg.n - 1 - c.i3 + sg.p);
    const int nvalid = (e_hi - e_lo + 1) * (o_hi - o_lo + 1);
    const bool producer = threadIdx.x == 0;
    const int row0 = static_cast<int>(sg.n * c.line_a);
    int pe = e_lo, po = o_lo, kp = 0;  // producer cursor: next step to load, its ring index
    auto produce = [&]() {             // loads of step (pe, po) into stage kp % nst
        const int st = kp % nst;
        const bool va = pe < sg.W, vb = pe >= 1;
        const int nbl = (c.i2 - sg.p + pe) + (sg.d < 3 ? 0 : sg.n * (c.i3 - sg.p + po));
        if (kp >= nst) mb_wait(empty + st, ((kp / nst) - 1) & 1);
        mb_expect(full + st, 8u * (sg.boxt * sg.LDR + 2 * ((va ? 1 : 0) + (vb ? 1 : 0)) * sg.W * sg.BR));
        tma3(su32(xs + st * sg.xstage), &mapX, -sg.p - sg.shift, nbl, c.t0, full + st);
        double* b0 = bsm + st * 4 * sg.bstage;
        if (va) {
            tma2(su32(b0), &mapM, row0, sg.W * (pe + sg.W * po), full + st);
            tma2(su32(b0 + 2 * sg.bstage), &mapK, row0, sg.W * (pe + sg.W * po), full + st);
        }
        if (vb) {
            tma2(su32(b0 + sg.bstage), &mapM, row0 + sg.n, sg.W * (pe - 1 + sg.W * po), full + st);
            tma2(su32(b0 + 3 * sg.bstage), &mapK, row0 + sg.n, sg.W * (pe - 1 + sg.W * po), full + st);
        }
        if (++pe > e_hi) {
            pe = e_lo;
            ++po;
        }
        ++kp;
    };
    if (producer)
        for (int i = 0; i < nst - 1 && kp < nvalid; ++i) produce();
    const int nwm = nwc / 2, wi = warp % nwm, mat = warp / nwm;
    const int ntiles = (c.tcols + 7) >> 3;
    double acc[RBW][kTT][2];
#pragma unroll
    for (int r = 0; r < RBW; ++r)
#pragma unroll
        for (int t = 0; t < kTT; ++t) acc[r][t][0] = acc[r][t][1] = 0.0;
    const int nr = min(RBW, sg.nblk - wi * RBW);  // live row blocks of this warp (<= 0: none)
    int ce = e_lo, st = 0, ph = 0;  // consumer cursor: offset e of step k, its stage and mbarrier phase
    for (int k = 0; k < nvalid; ++k) {
        if (producer && kp < nvalid) produce();  // step k + nst - 1 (waits until every warp released step k - 1)
        __syncwarp();
        const bool va = ce < sg.W, vb = ce >= 1;
        mb_wait(full + st, ph);
        const double* xst = xs + st * sg.xstage;
        const double* bm = bsm + (st * 4 + 2 * mat) * sg.bstage;
        if (nr == RBW && ntiles == kTT) {  // the usual case: every row block and time tile live
            pair_step_all<KS, RBW, RBW, true>(sg, xst, bm, wi * RBW, va, vb, ntiles, acc);
        } else {
#pragma unroll
            for (int r = 0; r < RBW; ++r) {
                if (r < nr) {
                    if (ntiles == kTT) pair_step_t<KS, true>(sg, xst, bm, wi * RBW + r, va, vb, ntiles, acc[r]);
                    else pair_step_t<KS, false>(sg, xst, bm, wi * RBW + r, va, vb, ntiles, acc[r]);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mb_arrive(empty + st);
        if (++ce > e_hi) ce = e_lo;
        if (++st == nst) {
            st = 0;
            ph ^= 1;
        }
    }
    const int g = lane >> 2, t4 = lane & 3;
    double* Y = mat ? KX : MX;
#pragma unroll
    for (int r = 0; r < RBW; ++r) {
        const int i1 = 4 * (wi * RBW + r) + (g & 3);
        if (i1 >= sg.n) continue;
        const long long irow = i1 + sg.n * (c.line_a + (g >> 2));
#pragma unroll
        for (int tt = 0; tt < kTT; ++tt)
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                const int tc = 8 * tt + 2 * t4 + v;
                if (tc < c.tcols) Y[irow + sg.Ns * (c.t0 + tc)] = acc[r][tt][v];
            }
    }
}

// (b) cp.async staging by all threads (warp = column group, lane = rows), double buffered.
template <int KS>
__global__ void __launch_bounds__(32 * 2 * kMaxWarps)
    stencil_sync_kernel(StencilGeo sg, const double* __restrict__ Mst, const double* __restrict__ Kst,
                        const double* __restrict__ X, double* __restrict__ MX, double* __restrict__ KX) {
    extern __shared__ __align__(128) double sx[];
    double* xs = sx;                   // 2 x xstage
    double* bsm = xs + 2 * sg.xstage;  // 2 x (M, K) x bstage
    const int nw = blockDim.x / 32;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const LineCtx c = line_ctx(sg);
    const int rows_seg = min(sg.seg_rows, sg.n - c.seg0);
    auto issue = [&](int s, long long nl, int buf) {
        const double* src = X + (c.seg0 - sg.p) + sg.n * nl + sg.Ns * c.t0;
        const unsigned dst = su32(xs + buf * sg.xstage);
        for (int col = warp; col < c.tcols; col += nw) {
            const double* sc = src + sg.Ns * col;
            const unsigned dc = dst + 8u * col * sg.LDR;
            for (int r = lane; r < sg.SR; r += 32) {
                const int j1 = c.seg0 - sg.p + r;
                const bool v = j1 >= 0 && j1 < sg.n;
                scp8(dc + 8u * r, v ? sc + r : X, v);
            }
        }
        const long long row0 = c.seg0 + sg.n * c.line;
        for (int mo = warp; mo < 2 * sg.W; mo += nw) {
            const int mat = mo / sg.W, o1 = mo - mat * sg.W;
            const double* bsrc = (mat ? Kst : Mst) + (o1 + static_cast<long long>(sg.W) * s) * sg.Ns + row0;
            const unsigned bd = su32(bsm + (buf * 2 + mat) * sg.bstage + o1 * sg.BR);
            for (int r = lane; r < sg.seg_rows; r += 32) scp8(bd + 8u * r, r < rows_seg ? bsrc + r : X, r < rows_seg);
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    const int nrb = nw / 2, rb = warp % nrb, mat = warp / nrb;
    const int ntiles = (c.tcols + 7) >> 3;
    double acc[kTT][2];
#pragma unroll
    for (int t = 0; t < kTT; ++t) acc[t][0] = acc[t][1] = 0.0;
    StepIter it(sg, c);
    if (it.valid()) issue(it.step(), it.line(), 0);
    int buf = 0;
    while (it.valid()) {
        it.next();
        asm volatile("cp.async.wait_group 0;\n" ::);
        __syncthreads();  // stage buf landed for all; the other buffer is free again
        if (it.valid()) issue(it.step(), it.line(), buf ^ 1);
        stencil_step<KS>(sg, xs + buf * sg.xstage, bsm + (buf * 2 + mat) * sg.bstage, rb, ntiles, acc);
        buf ^= 1;
    }
    stencil_store(sg, c, rb, acc, mat ? KX : MX);
}

template <int D>
__global__ void stencil_diag_kernel(PhysicalDesc g, const double* Kst, const double* Mst, double* dK, double* dM) {
    long long Ns = 1, c = 0, o = 1;
    for (int l = 0; l < D; ++l) {
        Ns *= g.n;
        c += g.p * o;
        o *= 2 * g.p + 1;
    }
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < Ns;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        dK[i] = Kst[c * Ns + i];
        dM[i] = Mst[c * Ns + i];
    }
}

template <int D>
cudaError_t assembly_d(const PhysicalDesc& g, double* Kst, double* Mst, cudaStream_t st) {
    long long elems = 1;
    int QD = 1;
    for (int l = 0; l < D; ++l) {
        elems *= g.n_el;
        QD *= g.q;
    }
    constexpr int NG = D * (D + 1) / 2 + 1;
    const size_t smem = sizeof(double) * (QD * NG + 2 * D * g.q * (g.p + 1)) + sizeof(int) * D;
    cudaError_t e = cudaFuncSetAttribute(physical_assembly_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    physical_assembly_kernel<D><<<static_cast<unsigned>(elems), 256, smem, st>>>(g, Kst, Mst);
    return cudaGetLastError();
}

template <int KS>
cudaError_t stencil_launch(const StencilGeo& sg, bool tma, dim3 grid, int nwc, const double* Mst, const double* Kst,
                           const double* X, const CUtensorMap* maps, double* MX, double* KX, cudaStream_t st) {
    if (tma) {
        const size_t smem = sizeof(double) * sg.nst * (sg.xstage + 2 * sg.bstage) + 2 * sg.nst * sizeof(uint64_t);
        cudaError_t e = cudaFuncSetAttribute(stencil_tma_kernel<KS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        stencil_tma_kernel<KS><<<grid, 32 * (2 * nwc + 1), smem, st>>>(sg, maps[0], maps[1], maps[2], MX, KX);
    } else {
        const size_t smem = sizeof(double) * 2 * (sg.xstage + 2 * sg.bstage);
        cudaError_t e = cudaFuncSetAttribute(stencil_sync_kernel<KS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(smem));
        if (e != cudaSuccess) return e;
        stencil_sync_kernel<KS><<<grid, 64 * nwc, smem, st>>>(sg, Mst, Kst, X, MX, KX);
    }
    return cudaGetLastError();
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
        cudaGetLastError();
    }
    return fn;
}

bool encode(CUtensorMap* m, const double* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
            const cuuint32_t* box) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return false;
    const cuuint32_t es[3] = {1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double*>(base), dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

cudaError_t launch_physical_assembly(const PhysicalDesc& g, double* Kst, double* Mst, cudaStream_t st) {
    if (g.p > kMaxP || g.pg > kMaxP) return cudaErrorInvalidValue;
    switch (g.d) {
        case 1: return assembly_d<1>(g, Kst, Mst, st);
        case 2: return assembly_d<2>(g, Kst, Mst, st);
        case 3: return assembly_d<3>(g, Kst, Mst, st);
        default: return cudaErrorInvalidValue;
    }
}

template <int KS, int RBW>
cudaError_t pair_launch(const PairGeo& sg, dim3 grid, const CUtensorMap* maps, double* MX, double* KX, cudaStream_t st) {
    const size_t smem = sizeof(double) * sg.nst * (sg.xstage + 4 * sg.bstage) + 2 * sg.nst * sizeof(uint64_t);
    cudaError_t e = cudaFuncSetAttribute(stencil_pair_kernel<KS, RBW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const int nwm = (sg.nblk + RBW - 1) / RBW;
    stencil_pair_kernel<KS, RBW><<<grid, 32 * 2 * nwm, smem, st>>>(sg, maps[0], maps[1], maps[2], MX, KX);
    return cudaGetLastError();
}

// Line-pair brick path (kernel (c)); returns cudaErrorNotSupported when the shape is not eligible.
cudaError_t launch_stencil_pair(const PhysicalDesc& g, const double* Mst, const double* Kst, const double* X, double* MX,
                                double* KX, long long n_t, cudaStream_t st) {
    if (g.d < 2 || g.n % 2 != 0 || (g.n + 3) / 4 > 18 || std::getenv("STIGA_STENCIL_NO_TMA") ||
        std::getenv("STIGA_STENCIL_NO_PAIR"))
        return cudaErrorNotSupported;
    if (((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Mst) | reinterpret_cast<uintptr_t>(Kst)) & 15u) != 0)
        return cudaErrorNotSupported;
    PairGeo sg;
    sg.n = g.n;
    sg.p = g.p;
    sg.W = 2 * g.p + 1;
    sg.d = g.d;
    sg.Ns = 1;
    long long pairs = g.n / 2;
    sg.nsteps = sg.W + 1;
    for (int l = 0; l < g.d; ++l) sg.Ns *= g.n;
    for (int l = 2; l < g.d; ++l) {
        pairs *= g.n;
        sg.nsteps *= sg.W;
    }
    sg.n_t = static_cast<int>(n_t);
    sg.nblk = (g.n + 3) / 4;
    const int KS = (4 + 2 * g.p + 3) / 4;
    sg.shift = g.p & 1;  // TMA boxes start on an even row
    const int SR = 4 * (sg.nblk - 1) + 4 * KS + sg.shift;
    sg.LDR = (SR + 11) / 16 * 16 + 4;
    if (sg.LDR - 16 >= SR) sg.LDR -= 16;
    sg.BR = (4 * sg.nblk + 11) / 16 * 16 + 4;
    if (sg.BR - 16 >= 4 * sg.nblk) sg.BR -= 16;
    sg.boxt = static_cast<int>(std::min<long long>(8 * kTT, n_t));
    sg.xstage = (sg.boxt * sg.LDR + 15) / 16 * 16;
    sg.bstage = (sg.W * sg.BR + 15) / 16 * 16;
    const size_t per = sizeof(double) * (sg.xstage + 4 * sg.bstage) + 2 * sizeof(uint64_t);
    sg.nst = static_cast<int>(std::min<size_t>(4, (227 * 1024) / per));
    if (sg.nst < 2 || sg.LDR > 256 || sg.BR > 256) return cudaErrorNotSupported;
    CUtensorMap maps[3];
    const cuuint64_t dx[3] = {static_cast<cuuint64_t>(g.n), static_cast<cuuint64_t>(sg.Ns / g.n),
                              static_cast<cuuint64_t>(n_t)};
    const cuuint64_t sx[2] = {static_cast<cuuint64_t>(g.n) * 8, static_cast<cuuint64_t>(sg.Ns) * 8};
    const cuuint32_t bx[3] = {static_cast<cuuint32_t>(sg.LDR), 1, static_cast<cuuint32_t>(sg.boxt)};
    long long planes = 1;
    for (int l = 0; l < g.d; ++l) planes *= sg.W;
    const cuuint64_t db[2] = {static_cast<cuuint64_t>(sg.Ns), static_cast<cuuint64_t>(planes)};
    const cuuint64_t sb[1] = {static_cast<cuuint64_t>(sg.Ns) * 8};
    const cuuint32_t bb[2] = {static_cast<cuuint32_t>(sg.BR), static_cast<cuuint32_t>(sg.W)};
    if (!(encode(&maps[0], X, 3, dx, sx, bx) && encode(&maps[1], Mst, 2, db, sb, bb) &&
          encode(&maps[2], Kst, 2, db, sb, bb)))
        return cudaErrorNotSupported;
    dim3 grid(static_cast<unsigned>(pairs), static_cast<unsigned>((n_t + 8 * kTT - 1) / (8 * kTT)));
#define STIGA_PAIR(KS_) \
    case KS_: return pair_launch<KS_, 3>(sg, grid, maps, MX, KX, st);
    switch (KS) {
        STIGA_PAIR(2)
        STIGA_PAIR(3)
        STIGA_PAIR(4)
        default: return cudaErrorNotSupported;
    }
#undef STIGA_PAIR
}

cudaError_t launch_stencil_apply2(const PhysicalDesc& g, const double* Mst, const double* Kst, const double* X,
                                  double* MX, double* KX, long long n_t, cudaStream_t st) {
    if (g.d < 1 || g.d > 3 || g.n <= 0 || n_t <= 0) return cudaErrorInvalidValue;
    {
        const cudaError_t pe = launch_stencil_pair(g, Mst, Kst, X, MX, KX, n_t, st);
        if (pe != cudaErrorNotSupported) return pe;
        if (std::getenv("STIGA_STENCIL_REQUIRE_PAIR")) return cudaErrorInvalidValue;  // tests: no silent fallback
    }
    StencilGeo sg;
    sg.n = g.n;
    sg.p = g.p;
    sg.W = 2 * g.p + 1;
    sg.d = g.d;
    sg.Ns = 1;
    long long lines = 1;
    sg.nsteps = 1;
    for (int l = 0; l < g.d; ++l) sg.Ns *= g.n;
    for (int l = 1; l < g.d; ++l) {
        lines *= g.n;
        sg.nsteps *= sg.W;
    }
    sg.n_t = static_cast<int>(n_t);
    const int KS = (8 + 2 * g.p + 3) / 4;
    const int blocks8 = (g.n + 7) / 8;
    sg.nseg = (blocks8 + kMaxWarps - 1) / kMaxWarps;
    const int wpc = (blocks8 + sg.nseg - 1) / sg.nseg;  // warps (row blocks) per segment
    sg.seg_rows = 8 * wpc;
    sg.SR = 8 * wpc - 8 + 4 * KS;
    // TMA boxes start on an even row: a box at an odd (negative) start coordinate faults, so odd p
    // stages one extra leading row
    const int shift = g.p & 1;
    sg.LDR = (sg.SR + shift + 11) / 16 * 16 + 4;
    if (sg.LDR - 16 >= sg.SR + shift) sg.LDR -= 16;
    sg.BR = (sg.seg_rows + 11) / 16 * 16 + 4;  // == 4 mod 16: conflict-free band fragments
    if (sg.BR - 16 >= sg.seg_rows) sg.BR -= 16;
    sg.xstage = (8 * kTT * sg.LDR + 15) / 16 * 16;
    sg.bstage = (sg.W * sg.BR + 15) / 16 * 16;
    sg.boxt = static_cast<int>(std::min<long long>(8 * kTT, n_t));
    sg.nst = kStages;
    dim3 grid(static_cast<unsigned>(lines * sg.nseg), static_cast<unsigned>((n_t + 8 * kTT - 1) / (8 * kTT)));
    // TMA staging needs 16-byte strides / base addresses (n even) and boxes <= 256 per dimension
    CUtensorMap maps[3];
    bool tma = g.n % 2 == 0 && sg.LDR <= 256 && sg.W <= 256 && sg.BR <= 256 && !std::getenv("STIGA_STENCIL_NO_TMA") &&
               ((reinterpret_cast<uintptr_t>(X) | reinterpret_cast<uintptr_t>(Mst) | reinterpret_cast<uintptr_t>(Kst)) &
                15u) == 0;
    if (tma) {
        const cuuint64_t dx[3] = {static_cast<cuuint64_t>(g.n), static_cast<cuuint64_t>(sg.Ns / g.n),
                                  static_cast<cuuint64_t>(n_t)};
        const cuuint64_t sx[2] = {static_cast<cuuint64_t>(g.n) * 8, static_cast<cuuint64_t>(sg.Ns) * 8};
        const cuuint32_t bx[3] = {static_cast<cuuint32_t>(sg.LDR), 1, static_cast<cuuint32_t>(sg.boxt)};
        long long planes = 1;
        for (int l = 0; l < g.d; ++l) planes *= sg.W;
        const cuuint64_t db[2] = {static_cast<cuuint64_t>(sg.Ns), static_cast<cuuint64_t>(planes)};
        const cuuint64_t sb[1] = {static_cast<cuuint64_t>(sg.Ns) * 8};
        const cuuint32_t bb[2] = {static_cast<cuuint32_t>(sg.BR), static_cast<cuuint32_t>(sg.W)};
        tma = encode(&maps[0], X, 3, dx, sx, bx) && encode(&maps[1], Mst, 2, db, sb, bb) &&
              encode(&maps[2], Kst, 2, db, sb, bb);
    }
    sg.shift = tma ? shift : 0;
    if (tma) {  // deepest ring that fits: X boxes of boxt columns (columns past n_t are never stored)
        sg.xstage = (sg.boxt * sg.LDR + 15) / 16 * 16;
        const size_t per = sizeof(double) * (sg.xstage + 2 * sg.bstage) + 2 * sizeof(uint64_t);
        sg.nst = static_cast<int>(std::min<size_t>(4, (227 * 1024) / per));
        if (sg.nst < 2) tma = false;
    }
    if (!tma) {
        sg.xstage = (8 * kTT * sg.LDR + 15) / 16 * 16;
        sg.shift = 0;
    }
    switch (KS) {
        case 3: return stencil_launch<3>(sg, tma, grid, wpc, Mst, Kst, X, maps, MX, KX, st);
        case 4: return stencil_launch<4>(sg, tma, grid, wpc, Mst, Kst, X, maps, MX, KX, st);
        case 5: return stencil_launch<5>(sg, tma, grid, wpc, Mst, Kst, X, maps, MX, KX, st);
        case 6: return stencil_launch<6>(sg, tma, grid, wpc, Mst, Kst, X, maps, MX, KX, st);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_stencil_diag(const PhysicalDesc& g, const double* Kst, const double* Mst, double* dK, double* dM,
                                cudaStream_t st) {
    const unsigned blocks = 148 * 8;
    switch (g.d) {
        case 1: stencil_diag_kernel<1><<<blocks, 256, 0, st>>>(g, Kst, Mst, dK, dM); break;
        case 2: stencil_diag_kernel<2><<<blocks, 256, 0, st>>>(g, Kst, Mst, dK, dM); break;
        case 3: stencil_diag_kernel<3><<<blocks, 256, 0, st>>>(g, Kst, Mst, dK, dM); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

}  // namespace gpu
}  // namespace stiga
