// Microbenchmark: DMMA m8n8k4 fed from shared memory with the fragment pattern of fd_kernels.cu.
// Measures the inner-loop ceiling (no global traffic) for several warp tilings.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kLDJ = 20;
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int MI, int NI, bool DB>
__global__ void probe(double* out, int iters, int WM, int LDX) {
  extern __shared__ double sm[];
  double* Js = sm; double* Xs = sm + MI * 8 * WM * kLDJ;
  for (int i = threadIdx.x; i < MI*8*WM*kLDJ + 16*LDX; i += blockDim.x) sm[i] = 1e-3 * (i % 7);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, wm = warp % WM, wn = warp / WM;
  const int g = lane >> 2, t = lane & 3;
  const double* ja = Js + (wm*MI*8 + g)*kLDJ + t;
  const double* bb = Xs + t*LDX + wn*NI*8 + g;
  double acc[MI][NI][2] = {};
  for (int it = 0; it < iters; ++it) {
    if (DB) {
      double av[2][MI], bv[2][NI];
      #pragma unroll
      for (int mi = 0; mi < MI; ++mi) av[0][mi] = ja[mi*8*kLDJ];
      #pragma unroll
      for (int ni = 0; ni < NI; ++ni) bv[0][ni] = bb[ni*8];
      #pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const int cur = kk & 1, nxt = cur ^ 1;
        if (kk + 1 < 4) {
          #pragma unroll
          for (int mi = 0; mi < MI; ++mi) av[nxt][mi] = ja[mi*8*kLDJ + (kk+1)*4];
          #pragma unroll
          for (int ni = 0; ni < NI; ++ni) bv[nxt][ni] = bb[(kk+1)*4*LDX + ni*8];
        }
        #pragma unroll
        for (int mi = 0; mi < MI; ++mi)
          #pragma unroll
          for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], av[cur][mi], bv[cur][ni]);
      }
    } else {
      #pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        double av[MI], bv[NI];
        #pragma unroll
        for (int mi = 0; mi < MI; ++mi) av[mi] = ja[mi*8*kLDJ + kk*4];
        #pragma unroll
        for (int ni = 0; ni < NI; ++ni) bv[ni] = bb[kk*4*LDX + ni*8];
        #pragma unroll
        for (int mi = 0; mi < MI; ++mi)
          #pragma unroll
          for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], av[mi], bv[ni]);
      }
    }
    __syncthreads();
  }
  double s = 0; for (int mi = 0; mi < MI; ++mi) for (int ni = 0; ni < NI; ++ni) s += acc[mi][ni][0] + acc[mi][ni][1];
  if (s == 1234.5) out[0] = s;
}
template <int MI, int NI, bool DB>
void run(int WM, int WN, int ctas_per_sm) {
  double* d; cudaMalloc(&d, 8);
  const int LDX = 8*NI*WN + 4;
  size_t smem = (MI*8*WM*kLDJ + 16*LDX) * 8;
  auto k = probe<MI, NI, DB>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int threads = 32*WM*WN, iters = 2000;
  int grid = 148 * ctas_per_sm;
  k<<<grid, threads, smem>>>(d, 10, WM, LDX);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<<<grid, threads, smem>>>(d, iters, WM, LDX); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  int occ; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, threads, smem);
  double fl = 2.0*256*MI*NI*4.0*iters*(WM*WN)*grid;
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, k);
  printf("MI=%2d NI=%d DB=%d WM=%d WN=%d ctas/SM=%d (occ %d) regs=%d warps/SM=%d : %.2f TF/s  %s\n", MI, NI, DB, WM, WN, ctas_per_sm, occ, fa.numRegs, WM*WN*ctas_per_sm, fl/ms/1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}
int main() {
  run<11,2,false>(1,4,3); run<11,2,true>(1,4,3);
  run<11,2,false>(3,4,1); run<11,2,true>(3,4,1);
  run<13,2,false>(1,4,2); run<13,2,true>(1,4,2);
  run<9,2,true>(4,2,1);  run<9,2,false>(4,2,1);
  run<7,2,true>(1,4,4); run<7,2,true>(2,4,2);
  run<4,4,true>(1,4,4); run<4,4,false>(1,4,4); run<8,4,false>(1,4,2); run<6,4,false>(1,4,3);
  run<2,8,false>(1,4,4); run<4,2,false>(1,4,4); run<2,2,false>(1,8,4);
  run<11,2,false>(1,4,4); run<11,2,false>(1,8,2); run<11,2,false>(1,2,6);
  return 0;
}
