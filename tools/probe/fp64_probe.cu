// Phase-0 box probe: FP64 DFMA/DADD issue rate, fp64 streaming bandwidth, device attributes.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s at %d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void dadd_loop(double* out, int iters, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 += b; x1 += b; x2 += b; x3 += b; x4 += b; x5 += b; x6 += b; x7 += b;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void ddiv_loop(double* out, int iters, double b) {
  double x0 = threadIdx.x + 1.5, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < iters; ++i) {
    x0 = b / x0 + 1.0; x1 = b / x1 + 1.0; x2 = b / x2 + 1.0; x3 = b / x3 + 1.0;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}
__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int l2 = 0, smemOptin = 0, clk = 0; cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  cudaDeviceGetAttribute(&smemOptin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  size_t fr, tot; CK(cudaMemGetInfo(&fr, &tot));
  printf("{\"name\":\"%s\",\"sms\":%d,\"l2_bytes\":%d,\"smem_optin\":%d,\"clock_khz\":%d,\"mem_free\":%zu,\"mem_total\":%zu,\"regs_per_sm\":%d}\n",
         p.name, p.multiProcessorCount, l2, smemOptin, clk, fr, tot, p.regsPerMultiprocessor);
  double* out; CK(cudaMalloc(&out, 148 * 8 * 1024 * sizeof(double)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 4, threads = 512, iters = 20000;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double inst = (double)blocks * threads * iters * 64;
    printf("{\"probe\":\"dfma\",\"ms\":%.3f,\"thread_inst_per_s\":%.4e,\"tflops\":%.3f}\n", ms, inst / (ms * 1e-3), 2 * inst / (ms * 1e-3) / 1e12);
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); dadd_loop<<<blocks, threads>>>(out, iters, 1e-7); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double inst = (double)blocks * threads * iters * 64;
    printf("{\"probe\":\"dadd\",\"ms\":%.3f,\"thread_inst_per_s\":%.4e}\n", ms, inst / (ms * 1e-3));
  }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); ddiv_loop<<<blocks, threads>>>(out, 2000, 3.0); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)blocks * threads * 2000 * 4;
    printf("{\"probe\":\"ddiv\",\"ms\":%.3f,\"div_per_s\":%.4e}\n", ms, n / (ms * 1e-3));
  }
  size_t n = (size_t)1 << 28; double2 *a, *b;  // 4 GiB each
  CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16)); cudaMemset(a, 0, n * 16);
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0); copy_kernel<<<p.multiProcessorCount * 8, 512>>>(a, b, n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"probe\":\"copy_fp64x2\",\"ms\":%.3f,\"gbs\":%.1f}\n", ms, 2.0 * n * 16 / (ms * 1e-3) / 1e9);
  }
  return 0;
}
