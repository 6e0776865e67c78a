// Microbenchmark: FP64 DFMA and DMMA (mma.sync m8n8k4 f64) throughput on the
// current GPU. Used to derive the "alu" roofline peak reported by bench.py.
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double acc[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i) acc[i] = fma(acc[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += acc[i];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int ILP>
__global__ void dmma_loop(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[ILP][2];
#pragma unroll
  for (int i = 0; i < ILP; ++i) { c[i][0] = i; c[i][1] = -i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < ILP; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

__global__ void dsqrt_loop(double* out, int iters) {
  double x = 2.0 + threadIdx.x;
  for (int it = 0; it < iters; ++it) x = sqrt(x) + 1.5;
  if (x == 12345.678) out[0] = x;
}
__global__ void ddiv_loop(double* out, int iters) {
  double x = 2.0 + threadIdx.x;
  for (int it = 0; it < iters; ++it) x = 3.0 / x + 1.5;
  if (x == 12345.678) out[0] = x;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("gpu %s sms %d clock_khz %d\n", p.name, p.multiProcessorCount, clk);
  double* out; cudaMalloc(&out, 4096 * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int threads : {256, 512, 1024}) {
    int iters = 20000; int blocks = sms * 2;
    dfma_loop<8><<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
    cudaEventRecord(e0);
    dfma_loop<8><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flop = 2.0 * 8 * iters * (double)blocks * threads;
    printf("DFMA threads=%d: %.2f TFLOP/s (%.3f ms)\n", threads, flop / ms / 1e9, ms);
  }
  for (int threads : {128, 256, 512}) {
    int iters = 20000; int blocks = sms * 2;
    dmma_loop<4><<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    dmma_loop<4><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flop = 2.0 * 256 * 4 * iters * (double)blocks * (threads / 32);
    printf("DMMA threads=%d: %.2f TFLOP/s (%.3f ms)\n", threads, flop / ms / 1e9, ms);
  }
  {
    int iters = 100000;
    dsqrt_loop<<<1, 32>>>(out, 10);
    cudaEventRecord(e0); dsqrt_loop<<<1, 32>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("dsqrt+add latency: %.1f ns/iter\n", ms * 1e6 / iters);
    ddiv_loop<<<1, 32>>>(out, 10);
    cudaEventRecord(e0); ddiv_loop<<<1, 32>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("ddiv+add latency: %.1f ns/iter\n", ms * 1e6 / iters);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
