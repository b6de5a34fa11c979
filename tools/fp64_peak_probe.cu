#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[8];
  #pragma unroll
  for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int u = 0; u < 16; ++u)
      #pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
  if (s == 12345.678) out[0] = s;
}
__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 0.5;
  double c[8][2];
  for (int i = 0; i < 8; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int u = 0; u < 4; ++u)
    #pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
int main() {
  double* d; cudaMalloc(&d, 8);
  int dev; cudaGetDevice(&dev); cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount; printf("SMs %d clock %d\n", sms, p.clockRate);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
  for (int tpb : {256, 512}) for (int bps : {1, 2, 4}) {
    int iters = 20000;
    dfma_kernel<<<sms*bps, tpb>>>(d, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_kernel<<<sms*bps, tpb>>>(d, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 128 * iters * (double)tpb * sms * bps;
    printf("DFMA tpb %d bps %d: %.2f TF/s (%.2f ms)\n", tpb, bps, fl / ms / 1e9, ms);
    iters = 5000;
    dmma_kernel<<<sms*bps, tpb>>>(d, 100);
    cudaEventRecord(e0);
    dmma_kernel<<<sms*bps, tpb>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    fl = 2.0 * 256 * 32 * iters * (double)(tpb/32) * sms * bps;
    printf("DMMA tpb %d bps %d: %.2f TF/s (%.2f ms)\n", tpb, bps, fl / ms / 1e9, ms);
  }}
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
}
