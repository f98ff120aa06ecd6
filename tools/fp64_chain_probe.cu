// Latency of the fold's sequential EWMA step L = fl(fl(b o) + fl(a L)) on one lane (the fold's
// exact fallback), in three forms: the loop as written (observation re-read from shared memory
// each step), unrolled with the observations in registers, and a bare dependent DADD chain.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o /tmp/fp64p tools/fp64_chain_probe.cu
#include <cstdio>
#include <cstdint>

__global__ void k(const double* in, double* out, int n, long long* cyc, double b, double a) {
  __shared__ double buf[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) buf[i] = in[i];
  __syncthreads();
  if (threadIdx.x) return;
  double L = 1.0;
  long long t0 = clock64();
  for (int r = 0; r < n; ++r)
    for (int u = 0; u < 256; ++u) L = __dadd_rn(__dmul_rn(b, buf[u]), __dmul_rn(a, L));
  long long t1 = clock64();
  out[0] = L;
  double M = 1.0;
  for (int r = 0; r < n; ++r) {
#pragma unroll 8
    for (int u = 0; u < 256; ++u) M = __dadd_rn(__dmul_rn(b, buf[u]), __dmul_rn(a, M));
  }
  long long t2 = clock64();
  out[1] = M;
  double Z = 1.0;
  for (int r = 0; r < n * 256; ++r) Z = __dadd_rn(Z, b);
  long long t3 = clock64();
  out[2] = Z;
  cyc[0] = t1 - t0;
  cyc[1] = t2 - t1;
  cyc[2] = t3 - t2;
}

int main() {
  double h[256];
  for (int i = 0; i < 256; ++i) h[i] = 1.0 + i * 1e-3;
  double *din, *dout;
  long long* dc;
  cudaMalloc(&din, sizeof h);
  cudaMalloc(&dout, 64);
  cudaMalloc(&dc, 64);
  cudaMemcpy(din, h, sizeof h, cudaMemcpyHostToDevice);
  const int n = 16;
  k<<<1, 32>>>(din, dout, n, dc, 0.5, 0.5);
  k<<<1, 32>>>(din, dout, n, dc, 0.5, 0.5);
  long long c[3];
  cudaMemcpy(c, dc, sizeof c, cudaMemcpyDeviceToHost);
  printf("cycles per step: loop %.1f  unrolled %.1f  bare DADD chain %.1f\n", c[0] / (n * 256.0),
         c[1] / (n * 256.0), c[2] / (n * 256.0));
  return 0;
}
