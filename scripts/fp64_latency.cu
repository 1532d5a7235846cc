// Dependent-chain latency of fp64 DMUL / DFMA / DADD and fp32 FMUL on this GPU
// (diagnostic for the sequential f3 cumsum / f7 product chains).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 scripts/fp64_latency.cu -o /tmp/fp64_latency
#include <cstdio>
template <int OP>
__global__ void chain(double* out, double a, double b, long long* cyc) {
  double x = a;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 4096; ++i) {
    if (OP == 0) x = __dmul_rn(x, b);
    else if (OP == 1) x = __fma_rn(x, b, a);
    else x = __dadd_rn(x, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
__global__ void chainf(float* out, float a, float b, long long* cyc) {
  float x = a;
  long long t0 = clock64();
#pragma unroll 16
  for (int i = 0; i < 4096; ++i) x = __fmul_rn(x, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  double* o; float* of; long long* c; long long h;
  cudaMalloc(&o, 1024 * 8); cudaMalloc(&of, 1024 * 4); cudaMalloc(&c, 8);
  const char* names[3] = {"DMUL", "DFMA", "DADD"};
  for (int rep = 0; rep < 2; ++rep) {
    chain<0><<<1, 32>>>(o, 1.0, 0.999999, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("%s %.1f cycles/op\n", names[0], h / 4096.0);
    chain<1><<<1, 32>>>(o, 1.0, 0.999999, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("%s %.1f cycles/op\n", names[1], h / 4096.0);
    chain<2><<<1, 32>>>(o, 1.0, 0.999999, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("%s %.1f cycles/op\n", names[2], h / 4096.0);
    chainf<<<1, 32>>>(of, 1.0f, 0.999999f, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    if (rep) printf("FMUL %.1f cycles/op\n", h / 4096.0);
  }
  return 0;
}
