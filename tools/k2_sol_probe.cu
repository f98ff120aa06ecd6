// Speed-of-light probe for the K2 step shape: a kernel with K2f's exact I/O (per invocation
// slack double2 + avail/supply/min_batch/flags in, idx/code/fill i32 + obj/slack/wait f64 out,
// 2^20 invocations = 71.3 MB) but no decision work, launched back to back over 4 rotating
// input sets (286 MB > L2) like bench.py, with and without programmatic dependent launch.
// The per-step time is the practical floor a decision kernel of this shape can reach.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/k2_sol_probe tools/k2_sol_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

struct IO {
  const double2* slack;
  const int* avail;
  const int* supply;
  const int* mb;
  const unsigned* flags;
  int* idx;
  int* code;
  int* fill;
  double* obj;
  double* sl;
  double* wait;
  unsigned N;
};

__global__ void __launch_bounds__(512, 2) k_sol(IO io, int pdl) {
  if (pdl) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
  }
  const unsigned stride = gridDim.x * blockDim.x;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < io.N; i += stride) {
    const double2 s = __ldg(io.slack + i);
    const int a = __ldg(io.avail + i), b = __ldg(io.supply + i), m = __ldg(io.mb + i);
    const unsigned f = __ldg(io.flags + i);
    io.idx[i] = a ^ (int)f;
    io.code[i] = b;
    io.fill[i] = m;
    io.obj[i] = s.x;
    io.sl[i] = s.y;
    io.wait[i] = s.x - s.y;
  }
}

int main() {
  const unsigned N = 1u << 20;
  const int SETS = 4, STEPS = 64;
  IO io[SETS];
  for (int s = 0; s < SETS; ++s) {
    void* p;
    cudaMalloc(&p, 16ull * N); cudaMemset(p, 0, 16ull * N); io[s].slack = (const double2*)p;
    cudaMalloc(&p, 4ull * N); cudaMemset(p, 0, 4ull * N); io[s].avail = (const int*)p;
    cudaMalloc(&p, 4ull * N); cudaMemset(p, 0, 4ull * N); io[s].supply = (const int*)p;
    cudaMalloc(&p, 4ull * N); cudaMemset(p, 0, 4ull * N); io[s].mb = (const int*)p;
    cudaMalloc(&p, 4ull * N); cudaMemset(p, 0, 4ull * N); io[s].flags = (const unsigned*)p;
    cudaMalloc(&p, 4ull * N); io[s].idx = (int*)p;
    cudaMalloc(&p, 4ull * N); io[s].code = (int*)p;
    cudaMalloc(&p, 4ull * N); io[s].fill = (int*)p;
    cudaMalloc(&p, 8ull * N); io[s].obj = (double*)p;
    cudaMalloc(&p, 8ull * N); io[s].sl = (double*)p;
    cudaMalloc(&p, 8ull * N); io[s].wait = (double*)p;
    io[s].N = N;
  }
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double bytes = (double)N * (32 + 36);
  for (int pdl = 0; pdl < 2; ++pdl) {
    for (int blocks_per_sm = 1; blocks_per_sm <= 2; ++blocks_per_sm) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(sms * 2);
      cfg.blockDim = dim3(512);
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = pdl;
      if (blocks_per_sm == 1) cfg.gridDim = dim3(sms * 4);  // 4 x 512 per SM: more in flight
      for (int w = 0; w < 8; ++w) cudaLaunchKernelEx(&cfg, k_sol, io[w % SETS], pdl);
      cudaEventRecord(a, st);
      for (int k = 0; k < STEPS; ++k) cudaLaunchKernelEx(&cfg, k_sol, io[k % SETS], pdl);
      cudaEventRecord(b, st);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double us = 1e3 * ms / STEPS;
      printf("{\"probe\": \"k2_sol\", \"pdl\": %d, \"grid\": %d, \"block\": 512, \"us_per_step\": %.3f, "
             "\"GBps\": %.1f}\n", pdl, cfg.gridDim.x, us, bytes / us / 1e3);
    }
  }
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}
