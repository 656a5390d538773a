// PCIe duplex probe: copy-engine (cudaMemcpyAsync) vs zero-copy SM kernels
// (loads from / stores to mapped pinned host memory), alone and concurrent.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_zc pcie_zc.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void zc_copy(const double2 *__restrict__ src, double2 *__restrict__ dst, size_t n2) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  // 4 independent 16-byte loads in flight per thread
  for (; i + 3 * st < n2; i += 4 * st) {
    double2 a = src[i], b = src[i + st], c = src[i + 2 * st], d = src[i + 3 * st];
    dst[i] = a; dst[i + st] = b; dst[i + 2 * st] = c; dst[i + 3 * st] = d;
  }
  for (; i < n2; i += st) dst[i] = src[i];
}

int main() {
  const size_t n = 99228483ull + 1, bytes = n * 8, n2 = n / 2;
  double *hin, *hout, *din, *dout;
  cudaHostAlloc(&hin, bytes, cudaHostAllocMapped);
  cudaHostAlloc(&hout, bytes, cudaHostAllocMapped);
  cudaMalloc(&din, bytes);
  cudaMalloc(&dout, bytes);
  for (size_t i = 0; i < n; ++i) hin[i] = (double)(i % 977);
  cudaMemset(dout, 0, bytes);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double *dhin, *dhout;
  cudaHostGetDevicePointer(&dhin, hin, 0);
  cudaHostGetDevicePointer(&dhout, hout, 0);
  auto timeit = [&](const char *name, auto fn) {
    fn();
    cudaDeviceSynchronize();
    cudaEventRecord(e0, 0);
    for (int r = 0; r < 5; ++r) fn();
    cudaEventRecord(e1, 0);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-44s %7.2f ms  (%5.1f GB/s per direction)\n", name, ms / 5, bytes / (ms / 5 * 1e6));
  };
  // legacy default stream 0 waits for s1/s2 (blocking streams not used: make s1/s2 join via events)
  cudaEvent_t j1, j2;
  cudaEventCreateWithFlags(&j1, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&j2, cudaEventDisableTiming);
  auto join = [&]() {
    cudaEventRecord(j1, s1);
    cudaEventRecord(j2, s2);
    cudaStreamWaitEvent(0, j1, 0);
    cudaStreamWaitEvent(0, j2, 0);
  };
  auto fork = [&]() {
    cudaEventRecord(j1, 0);
    cudaStreamWaitEvent(s1, j1, 0);
    cudaStreamWaitEvent(s2, j1, 0);
  };
  timeit("CE H2D", [&] { fork(); cudaMemcpyAsync(din, hin, bytes, cudaMemcpyHostToDevice, s1); join(); });
  timeit("CE D2H", [&] { fork(); cudaMemcpyAsync(hout, dout, bytes, cudaMemcpyDeviceToHost, s2); join(); });
  timeit("CE both", [&] {
    fork();
    cudaMemcpyAsync(din, hin, bytes, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(hout, dout, bytes, cudaMemcpyDeviceToHost, s2);
    join();
  });
  for (int g : {16, 32, 64, 148}) {
    char nm[96];
    snprintf(nm, sizeof nm, "ZC H2D kernel %d CTAs", g);
    timeit(nm, [&] { fork(); zc_copy<<<g, 512, 0, s1>>>((const double2 *)dhin, (double2 *)din, n2); join(); });
    snprintf(nm, sizeof nm, "ZC D2H kernel %d CTAs", g);
    timeit(nm, [&] { fork(); zc_copy<<<g, 512, 0, s2>>>((const double2 *)dout, (double2 *)dhout, n2); join(); });
    snprintf(nm, sizeof nm, "CE H2D + ZC D2H kernel %d CTAs", g);
    timeit(nm, [&] {
      fork();
      cudaMemcpyAsync(din, hin, bytes, cudaMemcpyHostToDevice, s1);
      zc_copy<<<g, 512, 0, s2>>>((const double2 *)dout, (double2 *)dhout, n2);
      join();
    });
    snprintf(nm, sizeof nm, "ZC H2D kernel + CE D2H %d CTAs", g);
    timeit(nm, [&] {
      fork();
      zc_copy<<<g, 512, 0, s1>>>((const double2 *)dhin, (double2 *)din, n2);
      cudaMemcpyAsync(hout, dout, bytes, cudaMemcpyDeviceToHost, s2);
      join();
    });
    snprintf(nm, sizeof nm, "ZC both kernels %d CTAs each", g);
    timeit(nm, [&] {
      fork();
      zc_copy<<<g, 512, 0, s1>>>((const double2 *)dhin, (double2 *)din, n2);
      zc_copy<<<g, 512, 0, s2>>>((const double2 *)dout, (double2 *)dhout, n2);
      join();
    });
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
