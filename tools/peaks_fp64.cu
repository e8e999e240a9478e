// FP64 roofline denominators for this pool's B200: DFMA pipe, DMMA (mma.sync f64),
// cuBLAS DGEMM, HBM copy / read, FP64 exp and reciprocal throughput.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o peaks_fp64 peaks_fp64.cu -lcublas
#include <cstdio>
#include <cuda_runtime.h>
#include <cublas_v2.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) { c[k][0] = 0; c[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(c[k][0], c[k][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void exp_kernel(double* out, int iters) {
  double x = threadIdx.x * 1e-4, s = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { s += exp(-(x + k * 1e-3)); x += 1e-7; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void rcp_kernel(double* out, int iters) {
  double x = 1.0 + threadIdx.x * 1e-4, s = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) { s += 1.0 / (x + k); x += 1e-7; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void read_kernel(const double2* __restrict__ a, double* out, size_t n) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) { double2 v = a[i]; s += v.x + v.y; }
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int sms = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d", p.name, sms, p.l2CacheSize);
  double* out; CK(cudaMalloc(&out, sizeof(double) * 1 << 24));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  // DFMA
  {
    int blocks = sms * 8, threads = 256, iters = 4096;
    dfma_kernel<<<blocks, threads>>>(out, 16, 1.0000001, 1e-9);
    CK(cudaDeviceSynchronize());
    float best = 1e30;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters, 1.0000001, 1e-9); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 64 * iters * (double)blocks * threads;
    printf(", \"dfma_tflops\": %.3f", flops / best / 1e9);
  }
  // DMMA
  {
    int blocks = sms * 8, threads = 256, iters = 4096;
    dmma_kernel<<<blocks, threads>>>(out, 16);
    CK(cudaDeviceSynchronize());
    float best = 1e30;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)blocks * (threads / 32);
    printf(", \"dmma_tflops\": %.3f", flops / best / 1e9);
  }
  // exp / rcp throughput (ops/s)
  {
    int blocks = sms * 8, threads = 256, iters = 512;
    exp_kernel<<<blocks, threads>>>(out, 4); CK(cudaDeviceSynchronize());
    float best = 1e30;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0); exp_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf(", \"exp_gops\": %.3f", 8.0 * iters * blocks * threads / best / 1e6);
    rcp_kernel<<<blocks, threads>>>(out, 4); CK(cudaDeviceSynchronize());
    best = 1e30;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0); rcp_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf(", \"div_gops\": %.3f", 8.0 * iters * blocks * threads / best / 1e6);
  }
  // HBM copy/read, 2 GiB buffers
  {
    size_t bytes = (size_t)2 << 30; size_t n2 = bytes / 16;
    double2 *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
    cudaMemset(a, 0, bytes); cudaMemset(b, 0, bytes);
    float best = 1e30;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0); copy_kernel<<<sms * 8, 512>>>(a, b, n2); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
    }
    printf(", \"copy_gbs\": %.1f", 2.0 * bytes / best / 1e6);
    best = 1e30;
    for (int r = 0; r < 6; ++r) {
      cudaEventRecord(e0); read_kernel<<<sms * 8, 512>>>(a, out, n2); cudaEventRecord(e1);
      cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
    }
    printf(", \"read_gbs\": %.1f", 1.0 * bytes / best / 1e6);
    cudaFree(a); cudaFree(b);
  }
  // cuBLAS DGEMM
  {
    cublasHandle_t h; cublasCreate(&h);
    int shapes[3][3] = {{4096, 4096, 4096}, {512, 4000, 512}, {8192, 8192, 8192}};
    const char* names[3] = {"dgemm_4096", "dgemm_512x4000x512", "dgemm_8192"};
    for (int s = 0; s < 3; ++s) {
      int m = shapes[s][0], n = shapes[s][1], k = shapes[s][2];
      double *A, *B, *C; CK(cudaMalloc(&A, sizeof(double) * m * k)); CK(cudaMalloc(&B, sizeof(double) * k * n)); CK(cudaMalloc(&C, sizeof(double) * m * n));
      cudaMemset(A, 0, sizeof(double) * m * k); cudaMemset(B, 0, sizeof(double) * k * n);
      double al = 1, be = 0; float best = 1e30;
      for (int r = 0; r < 6; ++r) {
        cudaEventRecord(e0); cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, m, n, k, &al, A, m, B, k, &be, C, m); cudaEventRecord(e1);
        cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (r && ms < best) best = ms;
      }
      printf(", \"%s_tflops\": %.3f, \"%s_us\": %.1f", names[s], 2.0 * m * n * k / best / 1e9, names[s], best * 1e3);
      cudaFree(A); cudaFree(B); cudaFree(C);
    }
    cublasDestroy(h);
  }
  printf("}\n");
  return 0;
}
