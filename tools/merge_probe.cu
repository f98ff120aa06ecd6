// Micro-benchmark: the plan builder's pairwise run merge (merge_runs) on one CTA.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

template <class T, class Less>
__device__ T* merge_runs(T* src, T* dst, int* off, int* s_nr, int n, Less less) {
  while (*s_nr > 1) {
    const int nr = *s_nr;
    for (int g = threadIdx.x; g < n; g += blockDim.x) {
      int lo = 0, hi = nr;
      while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (off[mid] <= g) lo = mid; else hi = mid;
      }
      int r = lo;
      while (r + 1 < nr && off[r + 1] <= g) ++r;
      const T x = src[g];
      const int pr = r ^ 1;
      const int base = off[r & ~1];
      if (pr >= nr) { dst[g] = x; continue; }
      const int pb = off[pr], pn = off[pr + 1] - pb;
      int a = 0, b = pn;
      if (r & 1) {
        while (a < b) { const int mid = (a + b) >> 1; if (!less(x, src[pb + mid])) a = mid + 1; else b = mid; }
      } else {
        while (a < b) { const int mid = (a + b) >> 1; if (less(src[pb + mid], x)) a = mid + 1; else b = mid; }
      }
      dst[base + (g - off[r]) + a] = x;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int m = 0;
      for (int i = 0; i < nr; i += 2) off[m++] = off[i];
      off[m] = n;
      *s_nr = m;
    }
    __syncthreads();
    T* t = src; src = dst; dst = t;
  }
  return src;
}

__global__ void k(const uint64_t* keys, const int* offs, int nr, int n, uint32_t* out, long long* cyc) {
  __shared__ uint64_t K[1024];
  __shared__ uint32_t A[1024], B[1024];
  __shared__ int off[65], s_nr;
  for (int i = threadIdx.x; i < n; i += blockDim.x) { K[i] = keys[i]; A[i] = i; }
  if (threadIdx.x <= nr) off[threadIdx.x] = offs[threadIdx.x];
  if (threadIdx.x == 0) s_nr = nr;
  __syncthreads();
  long long t0 = clock64();
  uint32_t* R = merge_runs(A, B, off, &s_nr, n, [&](uint32_t x, uint32_t y) { return K[x] < K[y]; });
  long long t1 = clock64();
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = R[i];
  if (threadIdx.x == 0) *cyc = t1 - t0;
}


template <class T, class Less>
__device__ T* merge_runs2(T* src, T* dst, uint8_t* rs, uint8_t* rd, int* off, int nr0, int n, Less less) {
  int nr = nr0;
  // rs[g] = run of position g
  while (nr > 1) {
    for (int g = threadIdx.x; g < n; g += blockDim.x) {
      const int r = rs[g];
      const T x = src[g];
      const int pr = r ^ 1;
      const int base = off[r & ~1];
      if (pr >= nr) { dst[g] = x; rd[g] = (uint8_t)(r >> 1); continue; }
      const int pb = off[pr], pn = off[pr + 1] - pb;
      int a = 0;
      const bool right = r & 1;
      for (int step = 1 << (31 - __clz(max(pn, 1))); step > 0; step >>= 1) {
        const int c = a + step;
        if (c <= pn) {
          const T y = src[pb + c - 1];
          const bool take = right ? !less(x, y) : less(y, x);
          if (take) a = c;
        }
      }
      const int np = base + (g - off[r]) + a;
      dst[np] = x;
      rd[np] = (uint8_t)(r >> 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int m = 0;
      for (int i = 0; i < nr; i += 2) off[m++] = off[i];
      off[m] = n;
    }
    nr = (nr + 1) >> 1;
    __syncthreads();
    T* t = src; src = dst; dst = t;
    uint8_t* u = rs; rs = rd; rd = u;
  }
  return src;
}

__global__ void k2(const uint64_t* keys, const int* offs, int nr, int n, uint32_t* out, long long* cyc) {
  __shared__ uint64_t K[1024];
  __shared__ uint32_t A[1024], B[1024];
  __shared__ uint8_t RA[1024], RB[1024];
  __shared__ int off[65];
  for (int i = threadIdx.x; i < n; i += blockDim.x) { K[i] = keys[i]; A[i] = i; }
  if (threadIdx.x <= nr) off[threadIdx.x] = offs[threadIdx.x];
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) { int r = 0; while (r + 1 < nr && off[r + 1] <= i) ++r; RA[i] = r; }
  __syncthreads();
  long long t0 = clock64();
  uint32_t* R = merge_runs2(A, B, RA, RB, off, nr, n, [&](uint32_t x, uint32_t y) { return K[x] < K[y]; });
  long long t1 = clock64();
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = R[i];
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  const int nr = 32, n = 736;
  std::vector<uint64_t> keys(n);
  std::vector<int> offs(nr + 1);
  std::mt19937_64 rng(1);
  for (int r = 0; r <= nr; ++r) offs[r] = r * n / nr;
  for (int r = 0; r < nr; ++r) {
    std::vector<uint64_t> v(offs[r + 1] - offs[r]);
    for (auto& x : v) x = rng();
    std::sort(v.begin(), v.end());
    std::copy(v.begin(), v.end(), keys.begin() + offs[r]);
  }
  uint64_t* dk; int* doff; uint32_t* dout; long long* dcyc;
  cudaMalloc(&dk, 8 * n); cudaMalloc(&doff, 4 * (nr + 1)); cudaMalloc(&dout, 4 * n); cudaMalloc(&dcyc, 8);
  cudaMemcpy(dk, keys.data(), 8 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(doff, offs.data(), 4 * (nr + 1), cudaMemcpyHostToDevice);
  for (int threads : {1024, 256, 128}) {
    for (int it = 0; it < 3; ++it) k<<<1, threads>>>(dk, doff, nr, n, dout, dcyc);
    long long cyc; cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
    std::vector<uint32_t> out(n); cudaMemcpy(out.data(), dout, 4 * n, cudaMemcpyDeviceToHost);
    bool ok = true; for (int i = 1; i < n; ++i) ok &= keys[out[i - 1]] <= keys[out[i]];
    printf("threads %d: merge %lld cycles, sorted %d\n", threads, cyc, (int)ok);
    for (int it = 0; it < 3; ++it) k2<<<1, threads>>>(dk, doff, nr, n, dout, dcyc);
    cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(out.data(), dout, 4 * n, cudaMemcpyDeviceToHost);
    ok = true; for (int i = 1; i < n; ++i) ok &= keys[out[i - 1]] <= keys[out[i]];
    printf("threads %d: merge2 %lld cycles, sorted %d\n", threads, cyc, (int)ok);
  }
  return 0;
}
