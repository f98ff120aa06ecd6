// PCIe probe: copy-engine vs SM-initiated (zero-copy) reads / writes of pinned host memory.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pcie_zc_probe pcie_zc_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__global__ void rd(const T* __restrict__ p, size_t n, T* sink) {
  T acc{};
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    T v = p[i];
    if constexpr (sizeof(T) == 16) { acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w; }
    else acc ^= v;
  }
  if constexpr (sizeof(T) == 16) { if (acc.x == 0x12345 && acc.y == 7) *sink = acc; }
  else if (acc == (T)0x12345) *sink = acc;
}
template <typename T>
__global__ void wr(T* __restrict__ p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    T v{};
    if constexpr (sizeof(T) == 16) { v.x = (unsigned)i; } else v = (T)i;
    p[i] = v;
  }
}
// read 32 B/element and write 36 B/element like the decision kernel, with chosen widths
__global__ void rw4(const unsigned* __restrict__ in, size_t n_in_words, unsigned* __restrict__ out,
                    size_t n_out_words) {
  size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  unsigned acc = 0;
  for (size_t i = g; i < n_in_words; i += st) acc ^= in[i];
  for (size_t i = g; i < n_out_words; i += st) out[i] = acc + (unsigned)i;
}
__global__ void rw16(const uint4* __restrict__ in, size_t n_in, uint4* __restrict__ out, size_t n_out) {
  size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  unsigned acc = 0;
  size_t m = n_in > n_out ? n_in : n_out;
  for (size_t i = g; i < m; i += st) {
    if (i < n_in) { uint4 v = in[i]; acc ^= v.x ^ v.w; }
    if (i < n_out) out[i] = make_uint4(acc, (unsigned)i, 0, 0);
  }
}

int main() {
  const size_t IN = 32ull << 20, OUT = 36ull << 20;  // ~ 2^20 decisions
  void *hin, *hout, *din, *dout, *sink;
  cudaHostAlloc(&hin, IN, cudaHostAllocDefault);
  cudaHostAlloc(&hout, OUT, cudaHostAllocDefault);
  cudaMalloc(&din, IN);
  cudaMalloc(&dout, OUT);
  cudaMalloc(&sink, 64);
  cudaStream_t s1, s2;
  cudaStreamCreate(&s1);
  cudaStreamCreate(&s2);
  cudaEvent_t a, b, c, d;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventCreateWithFlags(&c, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&d, cudaEventDisableTiming);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto time = [&](auto fn, const char* name, double bytes) {
    for (int w = 0; w < 2; ++w) fn();
    cudaDeviceSynchronize();
    cudaEventRecord(a, s1);
    for (int r = 0; r < 5; ++r) fn();
    cudaEventRecord(b, s1);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ms /= 5;
    printf("%-40s %8.3f ms  %7.1f GB/s\n", name, ms, bytes / ms / 1e6);
  };
  time([&] { cudaMemcpyAsync(din, hin, IN, cudaMemcpyHostToDevice, s1); }, "memcpy H2D 32MB", IN);
  time([&] { cudaMemcpyAsync(hout, dout, OUT, cudaMemcpyDeviceToHost, s1); }, "memcpy D2H 36MB", OUT);
  time([&] {
    cudaEventRecord(c, s1);  // fork s2 off s1, join it back (the timing events stay on s1)
    cudaStreamWaitEvent(s2, c);
    cudaMemcpyAsync(din, hin, IN, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(hout, dout, OUT, cudaMemcpyDeviceToHost, s2);
    cudaEventRecord(d, s2);
    cudaStreamWaitEvent(s1, d);
  }, "memcpy H2D||D2H", IN + OUT);
  for (int blocks : {sms, 4 * sms}) {
    char nm[64];
    snprintf(nm, 64, "zc read u32 (%d blk)", blocks);
    time([&] { rd<unsigned><<<blocks, 1024, 0, s1>>>((const unsigned*)hin, IN / 4, (unsigned*)sink); }, nm, IN);
    snprintf(nm, 64, "zc read u64 (%d blk)", blocks);
    time([&] { rd<unsigned long long><<<blocks, 1024, 0, s1>>>((const unsigned long long*)hin, IN / 8, (unsigned long long*)sink); }, nm, IN);
    snprintf(nm, 64, "zc read uint4 (%d blk)", blocks);
    time([&] { rd<uint4><<<blocks, 1024, 0, s1>>>((const uint4*)hin, IN / 16, (uint4*)sink); }, nm, IN);
    snprintf(nm, 64, "zc write u32 (%d blk)", blocks);
    time([&] { wr<unsigned><<<blocks, 1024, 0, s1>>>((unsigned*)hout, OUT / 4); }, nm, OUT);
    snprintf(nm, 64, "zc write u64 (%d blk)", blocks);
    time([&] { wr<unsigned long long><<<blocks, 1024, 0, s1>>>((unsigned long long*)hout, OUT / 8); }, nm, OUT);
    snprintf(nm, 64, "zc write uint4 (%d blk)", blocks);
    time([&] { wr<uint4><<<blocks, 1024, 0, s1>>>((uint4*)hout, OUT / 16); }, nm, OUT);
    snprintf(nm, 64, "zc read+write u32 (%d blk)", blocks);
    time([&] { rw4<<<blocks, 1024, 0, s1>>>((const unsigned*)hin, IN / 4, (unsigned*)hout, OUT / 4); }, nm, IN + OUT);
    snprintf(nm, 64, "zc read+write uint4 interleaved (%d blk)", blocks);
    time([&] { rw16<<<blocks, 1024, 0, s1>>>((const uint4*)hin, IN / 16, (uint4*)hout, OUT / 16); }, nm, IN + OUT);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
