// probe_gtimer.cu -- the update granularity of %globaltimer on this GPU
// (the device timeline and payload spans are read from it).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_gtimer.cu -o tools/probe_gtimer
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <map>

__global__ void k(unsigned long long* out, int n) {
  unsigned long long prev, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prev));
  int c = 0;
  while (c < n) {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t != prev) { out[c++] = t - prev; prev = t; }
  }
}

int main() {
  const int n = 20000;
  unsigned long long* d;
  cudaMalloc(&d, n * 8);
  k<<<1, 1>>>(d, n);
  unsigned long long h[n];
  cudaMemcpy(h, d, n * 8, cudaMemcpyDeviceToHost);
  std::map<unsigned long long, int> hist;
  for (int i = 0; i < n; ++i) hist[h[i]]++;
  printf("globaltimer step histogram (ns: count), %d steps:\n", n);
  int shown = 0;
  for (auto& kv : hist) { if (shown++ < 12) printf("  %llu: %d\n", kv.first, kv.second); }
  return 0;
}
