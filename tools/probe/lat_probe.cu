// FP64 dependent-chain latency probe (cycles per dependent op, single warp).
#include <cstdio>
__global__ void lat(double* out, long long* cyc, int n, double a) {
  double x = threadIdx.x * 1e-3 + 1.0, y = x + 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = x + a; x = x + a; x = x + a; x = x + a; }
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) { y = y * a; y = y * a; y = y * a; y = y * a; }
  long long t2 = clock64();
  double z = x;
  for (int i = 0; i < n; ++i) { z = fma(z, a, 1e-9); z = fma(z, a, 1e-9); z = fma(z, a, 1e-9); z = fma(z, a, 1e-9); }
  long long t3 = clock64();
  double w = y;
  for (int i = 0; i < n; ++i) { w = 1.0 / (w + 1.0); }
  long long t4 = clock64();
  double v = z;
  for (int i = 0; i < n; ++i) { v = sqrt(v + 2.0); }
  long long t5 = clock64();
  double u = w;
  for (int i = 0; i < n; ++i) { u = (u < v) ? u + 1.0 : v; }
  long long t6 = clock64();
  out[threadIdx.x] = x + y + z + w + v + u;
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 1024 * 8); cudaMallocManaged(&c, 64);
  int n = 4096;
  for (int r = 0; r < 2; ++r) { lat<<<1, 32>>>(o, c, n, 1.0000001); cudaDeviceSynchronize(); }
  printf("{\"dadd_lat\":%.2f,\"dmul_lat\":%.2f,\"dfma_lat\":%.2f,\"ddiv_chain\":%.2f,\"dsqrt_chain\":%.2f,\"dsetp_sel_dadd\":%.2f}\n",
         c[0] / (4.0 * n), c[1] / (4.0 * n), c[2] / (4.0 * n), c[3] / (1.0 * n), c[4] / (1.0 * n), c[5] / (1.0 * n));
  return 0;
}
