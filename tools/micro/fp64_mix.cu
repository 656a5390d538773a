// Are DMMA (mma.sync f64) and DFMA separate pipes on B200?  Mixed loop.
#include <cstdio>
#include <cuda_runtime.h>
template <int NF, int NM>
__global__ void mix(double *out, int iters, double a, double b) {
  double x[NF > 0 ? NF : 1];
#pragma unroll
  for (int i = 0; i < NF; ++i) x[i] = threadIdx.x * 1e-3 + i;
  double fa = threadIdx.x * 1e-3, fb = 1.0 - threadIdx.x * 1e-4;
  double c[NM > 0 ? NM : 1][2];
#pragma unroll
  for (int i = 0; i < NM; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NM; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(fa), "d"(fb));
#pragma unroll
    for (int i = 0; i < NF; ++i) x[i] = fma(x[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NF; ++i) s += x[i];
#pragma unroll
  for (int i = 0; i < NM; ++i) s += c[i][0] + c[i][1];
  if (s == 1234.5) out[0] = s;
}
template <int NF, int NM>
void run(double *out, int sms) {
  const int iters = 20000, nt = 256, grid = sms * 4;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  mix<NF, NM><<<grid, nt>>>(out, iters, 0.999, 1e-3);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  mix<NF, NM><<<grid, nt>>>(out, iters, 0.999, 1e-3);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double warps = (double)grid * nt / 32;
  double fma_fl = 2.0 * NF * iters * warps * 32, mma_fl = 2.0 * 256 * NM * iters * warps;
  double t = ms * 1e-3;
  printf("NF=%2d NM=%d : dfma %.2f TF + dmma %.2f TF = %.2f TF  (%.3f ms)\n", NF, NM, fma_fl / t * 1e-12,
         mma_fl / t * 1e-12, (fma_fl + mma_fl) / t * 1e-12, ms);
}
int main() {
  double *out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<8, 0>(out, sms); run<0, 4>(out, sms); run<8, 1>(out, sms); run<8, 2>(out, sms); run<8, 4>(out, sms);
  run<16, 2>(out, sms); run<16, 4>(out, sms); run<4, 4>(out, sms); run<32, 4>(out, sms);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
