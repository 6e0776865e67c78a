// Throughput probe: warp shuffles vs shared-memory broadcast vs DFMA on one B200
// (16 warps per SM, 148 CTAs).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o shfl_probe shfl_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int IT = 4096;
__global__ void k_shfl(double* out, int salt) {
  double z = threadIdx.x * 1e-3 + salt;
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
#pragma unroll 4
  for (int j = 0; j < IT; ++j) {
    const double x = __shfl_sync(0xffffffffu, z, j & 31);
    acc += x;
    z = z * 0.999 + (lane == (j & 31) ? 1e-9 : 0.0);
  }
  if (acc == 12345.0) out[0] = acc;
}
__global__ void k_shfl_indep(double* out, int salt) {   // 4 independent shuffles per iteration
  double z0 = threadIdx.x * 1e-3 + salt, z1 = z0 + 1, z2 = z0 + 2, z3 = z0 + 3;
  double acc = 0.0;
#pragma unroll 4
  for (int j = 0; j < IT; ++j) {
    acc += __shfl_sync(0xffffffffu, z0, j & 31) + __shfl_sync(0xffffffffu, z1, (j + 1) & 31) +
           __shfl_sync(0xffffffffu, z2, (j + 2) & 31) + __shfl_sync(0xffffffffu, z3, (j + 3) & 31);
  }
  if (acc == 12345.0) out[0] = acc;
}
__global__ void k_lds(double* out, int salt) {
  __shared__ double s[16][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  s[w][lane] = threadIdx.x * 1e-3 + salt;
  __syncwarp();
  double acc = 0.0;
#pragma unroll 4
  for (int j = 0; j < IT; ++j) acc += s[w][(j + (int)acc) & 31];
  if (acc == 12345.0) out[0] = acc;
}
__global__ void k_lds_indep(double* out, int salt) {
  __shared__ double s[16][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  s[w][lane] = threadIdx.x * 1e-3 + salt;
  __syncwarp();
  volatile double* vs = s[w];
  double acc = 0.0;
#pragma unroll 4
  for (int j = 0; j < IT; ++j) acc += vs[j & 31] + vs[(j + 1) & 31] + vs[(j + 2) & 31] + vs[(j + 3) & 31];
  if (acc == 12345.0) out[0] = acc;
}
__global__ void k_lds_lane(double* out, int salt) {   // lane-distinct 8-byte loads (2 wavefronts each)
  __shared__ double s[16][64];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  s[w][lane] = s[w][lane + 32] = threadIdx.x * 1e-3 + salt;
  __syncwarp();
  volatile double* vs = s[w];
  double acc = 0.0;
#pragma unroll 4
  for (int j = 0; j < IT; ++j) acc += vs[(lane + j) & 63] + vs[(lane + j + 1) & 63] + vs[(lane + j + 2) & 63] + vs[(lane + j + 3) & 63];
  if (acc == 12345.0) out[0] = acc;
}
__global__ void k_dfma(double* out, int salt) {
  double a = threadIdx.x * 1e-3 + salt, b = a + 1, c = a + 2, d = a + 3;
#pragma unroll 4
  for (int j = 0; j < IT; ++j) {
    a = fma(a, 0.999, 1e-3); b = fma(b, 0.999, 1e-3); c = fma(c, 0.999, 1e-3); d = fma(d, 0.999, 1e-3);
  }
  if (a + b + c + d == 12345.0) out[0] = a;
}
template <typename K>
float run(K k, const char* name, int nops) {
  double* o;
  cudaMalloc(&o, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<148, 512>>>(o, 1);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<<<148, 512>>>(o, r);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= 5;
  const double cyc = ms * 1e-3 * 1.965e9;
  const double per_sm_ops = 16.0 * IT * nops;   // warp-instructions per SM
  printf("%-12s %.3f ms  %.2f SM-cycles per warp-op\n", name, ms, cyc / per_sm_ops);
  cudaFree(o);
  return ms;
}
int main() {
  run(k_shfl, "shfl_dep", 2);        // a 64-bit shuffle = 2 SHFL
  run(k_shfl_indep, "shfl_x4", 8);
  run(k_lds, "lds_bcast", 1);
  run(k_lds_indep, "lds_bc_x4", 4);
  run(k_lds_lane, "lds_lane_x4", 4);
  run(k_dfma, "dfma_x4", 4);
  return 0;
}
