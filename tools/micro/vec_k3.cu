// MINRES K3-style streaming update: which variant reaches HBM bandwidth?
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NT = 256;
template <int V>
__global__ void __launch_bounds__(NT) k3(long n, const double *__restrict__ z, double *__restrict__ v,
                                         const double *__restrict__ w, double *__restrict__ w1,
                                         const double *__restrict__ w2, double *__restrict__ x, double oldeps,
                                         double delta, double gamma, double phi, double beta) {
  if constexpr (V == 0 || V == 1) {
    const double rg = 1.0 / gamma, rb = 1.0 / beta;
    for (long i = (long)blockIdx.x * NT + threadIdx.x; i < n; i += (long)gridDim.x * NT) {
      const double vi = v[i];
      const double wn = V == 0 ? (vi - oldeps * w2[i] - delta * w[i]) / gamma : (vi - oldeps * w2[i] - delta * w[i]) * rg;
      w1[i] = wn;
      x[i] = x[i] + phi * wn;
      v[i] = V == 0 ? z[i] / beta : z[i] * rb;
    }
  } else {
    const long n2 = n / 2;
    const double2 *z2 = (const double2 *)z, *w22 = (const double2 *)w2, *ww = (const double2 *)w;
    double2 *v2 = (double2 *)v, *w12 = (double2 *)w1, *x2 = (double2 *)x;
    for (long i = (long)blockIdx.x * NT + threadIdx.x; i < n2; i += (long)gridDim.x * NT) {
      const double2 vi = v2[i], a = w22[i], b = ww[i], xx = x2[i], zz = z2[i];
      double2 wn, xo, vo;
      wn.x = (vi.x - oldeps * a.x - delta * b.x) / gamma;
      wn.y = (vi.y - oldeps * a.y - delta * b.y) / gamma;
      w12[i] = wn;
      xo.x = xx.x + phi * wn.x;
      xo.y = xx.y + phi * wn.y;
      x2[i] = xo;
      vo.x = zz.x / beta;
      vo.y = zz.y / beta;
      v2[i] = vo;
    }
  }
}
int main() {
  const long n = 99228483L + 1;
  double *b[6];
  for (int i = 0; i < 6; ++i) { cudaMalloc(&b[i], n * 8); cudaMemset(b[i], 0, n * 8); }
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int V = 0; V < 3; ++V)
    for (int mult : {4, 8, 16, 32}) {
      int grid = sms * mult;
      auto go = [&] {
        if (V == 0) k3<0><<<grid, NT>>>(n, b[0], b[1], b[2], b[3], b[4], b[5], 0.1, 0.2, 1.3, 0.4, 1.7);
        if (V == 1) k3<1><<<grid, NT>>>(n, b[0], b[1], b[2], b[3], b[4], b[5], 0.1, 0.2, 1.3, 0.4, 1.7);
        if (V == 2) k3<2><<<grid, NT>>>(n, b[0], b[1], b[2], b[3], b[4], b[5], 0.1, 0.2, 1.3, 0.4, 1.7);
      };
      go(); cudaDeviceSynchronize();
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) go();
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
      printf("V=%d grid=%dx%d: %.3f ms  %.0f GB/s\n", V, sms, mult, ms, 8.0 * 8 * n / ms / 1e6);
    }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
