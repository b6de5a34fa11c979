// A/B evidence for the DMMA-vs-DFMA choice of the FD mode products (north_star (2): "FP64 DMMA
// tensor-core tiles only where ncu shows they beat the FFMA path on these small n x n contractions").
//
// The same product the FD apply runs for its last (time) mode -- Y = J X with J (m x n, row-major)
// and X (n x N, N = number of fibers, contiguous along N; kronop.cpp:43-73 with L = N) -- on the
// FP64 CUDA cores: a register-tiled DFMA GEMM (thread tile TM x 4, CTA tile 8 TM x 128, k-chunks of
// 16 through a 3-stage 16-byte cp.async ring, A and B operands as LDS.128 (A: warp broadcasts), two
// CTAs per SM).
// Its launch time is compared with the product's DMMA kernel on the same shape (the autotuner's
// "[stiga tune] time gemm" lines, STIGA_DEBUG_TUNE=1) and both are profiled with ncu
// (sm__pipe_fp64_cycles_active, sm__pipe_tensor_subpipe_dmma_cycles_active).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o /tmp/dfma_probe tools/dfma_mode_probe.cu
//   /tmp/dfma_probe            # the BASELINE time-mode shapes: c4 67 x 287496, c3 98 x 912673, c2 258 x 66049
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cmath>
#include <cuda_runtime.h>

constexpr int BK = 16, BN = 128, NTHR = 256, NS = 3;

__device__ __forceinline__ void cp16(unsigned s, const double* g, bool valid) {
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(g), "r"(sz));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }

// Jt: Kp x Mp (k-major, zero padded: Mp = gridDim.y * 8 TM, Kp = multiple of 16); X: n x N; Y: m x N.
// Thread (tx, ty): rows r0 + TM ty .. + TM - 1 (a contiguous group, staged at pitch PT = TM rounded up
// to even so the A operand is read as 16-byte warp broadcasts), columns 4 tx .. 4 tx + 3.
template <int TM>
__global__ void __launch_bounds__(NTHR, 2) dfma_mode_kernel(const double* __restrict__ Jt, const double* __restrict__ X,
                                                         double* __restrict__ Y, int m, int n, int Kp, int Mp, long long N) {
  constexpr int BM = 8 * TM, PT = (TM + 1) & ~1, BMS = 8 * PT;
  extern __shared__ __align__(16) double sm[];
  double* As = sm;                  // NS x BK x BMS
  double* Bs = sm + NS * BK * BMS;  // NS x BK x BN
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = (lane & 7) + 8 * (warp & 3);   // 0..31: columns 4 tx .. 4 tx + 3
  const int ty = (lane >> 3) + 4 * (warp >> 2); // 0..7: rows ty + 8 i
  const long long c0 = static_cast<long long>(blockIdx.x) * BN;
  const int r0 = blockIdx.y * BM;
  const int nchunks = Kp / BK;
  auto issue = [&](int q, int st) {
    const int k0 = q * BK;
    // B chunk: 16 rows x 128 columns = 1024 16-byte pieces, 4 per thread
#pragma unroll
    for (int u = 0; u < BK * BN / 2 / NTHR; ++u) {
      const int piece = tid + u * NTHR, row = piece / (BN / 2), col = 2 * (piece % (BN / 2));
      const bool v = k0 + row < n && c0 + col < N;  // N even in every shape used here
      cp16(static_cast<unsigned>(__cvta_generic_to_shared(Bs + (st * BK + row) * BN + col)),
           v ? X + static_cast<long long>(k0 + row) * N + c0 + col : X, v);
    }
    // A chunk: 16 rows x 8 groups of PT (the global copy is padded the same way: Mp = gridDim.y * BMS)
    for (int piece = tid; piece < BK * BMS / 2; piece += NTHR) {
      const int row = piece / (BMS / 2), col = 2 * (piece % (BMS / 2));
      cp16(static_cast<unsigned>(__cvta_generic_to_shared(As + (st * BK + row) * BMS + col)),
           Jt + static_cast<long long>(k0 + row) * Mp + blockIdx.y * BMS + col, true);
    }
  };
  double acc[TM][4];
#pragma unroll
  for (int i = 0; i < TM; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.0;
  for (int s = 0; s < NS - 1; ++s) {
    if (s < nchunks) issue(s, s);
    cp_commit();
  }
  int st = 0;
  for (int q = 0; q < nchunks; ++q) {
    cp_wait1();
    __syncthreads();
    if (q + NS - 1 < nchunks) issue(q + NS - 1, (st + NS - 1) % NS);
    cp_commit();
    const double* a = As + st * BK * BMS + PT * ty;
    const double* b = Bs + st * BK * BN + 4 * tx;
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      const double2 b0 = *reinterpret_cast<const double2*>(b + k * BN);
      const double2 b1 = *reinterpret_cast<const double2*>(b + k * BN + 2);
      double av[PT];
#pragma unroll
      for (int i = 0; i < PT / 2; ++i) {
        const double2 a2 = *reinterpret_cast<const double2*>(a + k * BMS + 2 * i);
        av[2 * i] = a2.x;
        av[2 * i + 1] = a2.y;
      }
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        acc[i][0] = fma(av[i], b0.x, acc[i][0]);
        acc[i][1] = fma(av[i], b0.y, acc[i][1]);
        acc[i][2] = fma(av[i], b1.x, acc[i][2]);
        acc[i][3] = fma(av[i], b1.y, acc[i][3]);
      }
    }
    st = (st + 1) % NS;
  }
  const long long c = c0 + 4 * tx;
  if (c < N) {
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int r = r0 + TM * ty + i;
      if (r < m) {
        double* y = Y + static_cast<long long>(r) * N + c;
        *reinterpret_cast<double2*>(y) = make_double2(acc[i][0], acc[i][1]);
        *reinterpret_cast<double2*>(y + 2) = make_double2(acc[i][2], acc[i][3]);
      }
    }
  }
}

template <int TM>
float run(const double* Jt, const double* X, double* Y, int m, int n, int Kp, int rb, long long N, int reps) {
  auto k = dfma_mode_kernel<TM>;
  constexpr int PT = (TM + 1) & ~1;
  const size_t smem = sizeof(double) * NS * BK * (8 * PT + BN);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  dim3 grid(static_cast<unsigned>((N + BN - 1) / BN), rb);
  const int Mp = rb * 8 * PT;
  k<<<grid, NTHR, smem>>>(Jt, X, Y, m, n, Kp, Mp, N);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(e0);
    k<<<grid, NTHR, smem>>>(Jt, X, Y, m, n, Kp, Mp, N);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, NTHR, smem);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, k);
  std::printf("  DFMA TM=%2d row blocks=%d regs=%d ctas/SM=%d: %.4f ms  %.2f TF/s (2 m n N)  %s\n", TM, rb, fa.numRegs, occ, best,
              2.0 * m * n * static_cast<double>(N) / best / 1e9, cudaGetErrorString(cudaGetLastError()));
  return best;
}

void shape(const char* name, int n, long long N) {
  const int m = n;
  std::printf("%s: J %d x %d, %lld fibers (%.1f M DoF)\n", name, m, n, N, m * static_cast<double>(N) / 1e6);
  const int Kp = (n + BK - 1) / BK * BK;
  const int MpMax = 2 * 8 * 13 * 3;
  std::vector<double> J(static_cast<size_t>(m) * n), x(static_cast<size_t>(n) * 4096);
  unsigned long long s = 88172645463325252ull;
  auto rnd = [&] { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return (s >> 11) * (1.0 / 9007199254740992.0) * 2 - 1; };
  for (auto& v : J) v = rnd();
  double *dJt, *dX, *dY;
  cudaMalloc(&dJt, sizeof(double) * Kp * MpMax);
  cudaMalloc(&dX, sizeof(double) * n * N);
  cudaMalloc(&dY, sizeof(double) * m * N);
  // X: a 4096-column random block repeated (a device-side fill keeps the probe short)
  for (auto& v : x) v = rnd();
  for (int k = 0; k < n; ++k)
    for (long long c = 0; c < N; c += 4096) {
      const long long w = (N - c < 4096) ? N - c : 4096;
      cudaMemcpy(dX + static_cast<long long>(k) * N + c, x.data() + static_cast<size_t>(k) * 4096, sizeof(double) * w,
                 cudaMemcpyHostToDevice);
    }
  auto upload = [&](int TM, int RB) {  // row i -> block i / (8 TM), group (i % (8 TM)) / TM, slot i % TM at pitch PT
    const int PT = (TM + 1) & ~1, Mp = RB * 8 * PT;
    std::vector<double> Jt(static_cast<size_t>(Kp) * Mp, 0.0);
    for (int i = 0; i < m; ++i) {
      const int blk = i / (8 * TM), in = i % (8 * TM), pos = blk * 8 * PT + (in / TM) * PT + in % TM;
      for (int k = 0; k < n; ++k) Jt[static_cast<size_t>(k) * Mp + pos] = J[static_cast<size_t>(i) * n + k];
    }
    cudaMemcpy(dJt, Jt.data(), sizeof(double) * Jt.size(), cudaMemcpyHostToDevice);
  };
  auto check = [&] {  // column 5 and the last column against a host dot product
    double err = 0;
    for (long long c : {5LL, N - 1}) {
      std::vector<double> xc(n), yc(m);
      for (int k = 0; k < n; ++k) cudaMemcpy(&xc[k], dX + static_cast<long long>(k) * N + c, 8, cudaMemcpyDeviceToHost);
      for (int i = 0; i < m; ++i) cudaMemcpy(&yc[i], dY + static_cast<long long>(i) * N + c, 8, cudaMemcpyDeviceToHost);
      for (int i = 0; i < m; ++i) {
        double r = 0;
        for (int k = 0; k < n; ++k) r += J[static_cast<size_t>(i) * n + k] * xc[k];
        err = std::fmax(err, std::fabs(r - yc[i]));
      }
    }
    std::printf("  max |error| on two columns: %.2e\n", err);
  };
#define RUN(TM, RB)                                         \
  if (8 * TM * RB >= m && 8 * TM * RB - m < 16) {          \
    upload(TM, RB);                                         \
    cudaMemset(dY, 0, sizeof(double) * m * N);              \
    run<TM>(dJt, dX, dY, m, n, Kp, RB, N, 5);               \
    check();                                                \
  }
  RUN(9, 1) RUN(5, 2) RUN(13, 1) RUN(7, 2) RUN(11, 3) RUN(9, 4) RUN(12, 3)
#undef RUN
  cudaFree(dJt);
  cudaFree(dX);
  cudaFree(dY);
}

int main(int argc, char** argv) {
  if (argc == 3) {
    shape("custom", std::atoi(argv[1]), std::atoll(argv[2]));
    return 0;
  }
  shape("c4 time mode", 67, 287496);
  shape("c3 time mode", 98, 912673 - 1);  // even fiber count (16-byte rows)
  shape("c2 time mode", 258, 66049 - 1);
  return 0;
}
