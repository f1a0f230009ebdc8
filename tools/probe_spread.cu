// probe_spread.cu -- which direction carries the ~1 us spread of the host<->GPU
// round trip?  148 pollers, round robin; the target echoes the value and the
// %globaltimer at which it saw it.  The host<->device clock offset is
// constant, so the spread (p90 - p10) of each one-way leg is exact even
// though its mean is not.  (design probe, not product code)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_spread.cu -o tools/probe_spread
#include <cuda_runtime.h>
#include <immintrin.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <time.h>
#include <unistd.h>

#include <algorithm>
#include <vector>

static inline uint64_t now_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return uint64_t(ts.tv_sec) * 1000000000ull + ts.tv_nsec;
}
__device__ __forceinline__ unsigned long long ldr64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__global__ void pollers(const unsigned long long* flags, unsigned long long* echo, uint32_t last) {
  if (threadIdx.x) return;
  const unsigned long long* f = flags + 16 * blockIdx.x;
  unsigned long long* o = echo + 16 * blockIdx.x;
  unsigned long long seen = 0;
  for (;;) {
    const unsigned long long v = ldr64(f);
    if (v != seen) {
      const unsigned long long t = gtime();
      seen = v;
      asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(o), "l"(v), "l"(t) : "memory");
      if (v >= last) return;
    }
  }
}

static void stats(const char* label, std::vector<int64_t> v) {
  std::sort(v.begin(), v.end());
  const int64_t base = v[v.size() / 2];   // relative to the median: keeps double precision
  auto q = [&](double p) { return (v[size_t(p * (v.size() - 1))] - base) / 1e3; };
  printf("%-34s p10 %+7.3f p50 %+7.3f p90 %+7.3f us (about the median)  spread(p90-p10) %.3f us\n", label, q(0.1),
         q(0.5), q(0.9), q(0.9) - q(0.1));
}

int main() {
  cudaSetDevice(0);
  cudaFree(0);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const uint32_t R = 40000;
  unsigned long long* cells;
  const size_t bytes = size_t(nsm) * 128 * 2 + 4096;
  cudaHostAlloc(&cells, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int grid : {nsm, 1}) {
    memset(cells, 0, bytes);
    volatile unsigned long long* flags = cells;
    volatile unsigned long long* echo = cells + 16 * nsm + 512;
    pollers<<<grid, 32, 0, st>>>((const unsigned long long*)flags, (unsigned long long*)echo, R);
    usleep(2000);
    std::vector<int64_t> down, up, rt;
    bool bad = false;
    for (uint32_t r = 1; r <= R && !bad; ++r) {
      const uint32_t t = r % grid;
      const uint64_t t0 = now_ns();
      if (r == R) for (int i = 0; i < grid; ++i) flags[16 * i] = R;
      else flags[16 * t] = r;
      const uint64_t dl = t0 + 2000000000ull;
      while (echo[16 * t] != r) {
        _mm_pause();
        if (now_ns() > dl) { bad = true; break; }
      }
      const uint64_t t2 = now_ns();
      const int64_t d = int64_t(echo[16 * t + 1]);
      if (r > R / 10 && r < R) {
        down.push_back(d - int64_t(t0));
        up.push_back(int64_t(t2) - d);
        rt.push_back(int64_t(t2 - t0));
      }
    }
    cudaStreamSynchronize(st);
    if (bad) { printf("stalled\n"); continue; }
    // remove the unknown offset from the one-way legs: shift so their p50s add up to the round trip's p50
    printf("%d poller(s):\n", grid);
    stats("  round trip", rt);
    stats("  host write -> device sees (+off)", down);
    stats("  device sees -> host sees (-off)", up);
    fflush(stdout);
  }
  return 0;
}
