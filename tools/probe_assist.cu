// probe_assist.cu -- the HYBRID-style split: poller warps forward each new
// host-cell value into shared memory and a separate protocol warp, spinning
// on shared memory, echoes it.  1 or 2 poller warps (2 replica lines,
// started `spacing` apart) vs the poller echoing directly.  148 SMs, round
// robin.  Does the shared-memory hop cost anything, and does a second
// poller warp then pay?  (design probe, not product code)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_assist.cu -o tools/probe_assist
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
// mode 0: warp 0 polls line 0 and echoes.  mode 1: warp 1 polls line 0 ->
// smem; warp 0 spins on smem and echoes.  mode 2: warps 1 and 2 poll lines 0
// and 1 (spacing apart) -> smem; warp 0 echoes the newest.
__global__ void k(const unsigned long long* flags, unsigned long long* echo, uint32_t last, int mode, uint32_t sp) {
  __shared__ unsigned long long slot[2];
  __shared__ volatile uint32_t stop;
  if (threadIdx.x == 0) { slot[0] = slot[1] = 0; stop = 0; }
  __syncthreads();
  const uint32_t i = blockIdx.x, w = threadIdx.x >> 5;
  if (threadIdx.x & 31) return;
  const unsigned long long* line0 = flags + (i * 2) * 16;
  unsigned long long* o = echo + 16 * i;
  if (mode == 0) {
    if (w) return;
    unsigned long long seen = 0;
    for (;;) {
      const unsigned long long v = ldr64(line0);
      if (v > seen) {
        seen = v;
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(o), "l"(v) : "memory");
        if (v >= last) return;
      }
    }
  }
  const int npoll = mode == 1 ? 1 : 2;
  if (w >= 1 && int(w) <= npoll) {   // poller warps
    const unsigned long long* f = line0 + (w - 1) * 16;
    if (w == 2) __nanosleep(sp);
    unsigned long long seen = 0;
    while (!stop) {
      const unsigned long long v = ldr64(f);
      if (v > seen) {
        seen = v;
        *(volatile unsigned long long*)&slot[w - 1] = v;
      }
    }
    return;
  }
  if (w != 0) return;
  unsigned long long seen = 0;   // protocol warp
  for (;;) {
    const unsigned long long a = *(volatile unsigned long long*)&slot[0];
    const unsigned long long b = npoll == 2 ? *(volatile unsigned long long*)&slot[1] : 0;
    const unsigned long long v = a > b ? a : b;
    if (v > seen) {
      seen = v;
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(o), "l"(v) : "memory");
      if (v >= last) { stop = 1; return; }
    }
  }
}

int main() {
  cudaSetDevice(0);
  cudaFree(0);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const uint32_t R = 40000;
  unsigned long long* cells;
  const size_t bytes = size_t(nsm) * 128 * 3 + 4096;
  cudaHostAlloc(&cells, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  struct V { int mode; uint32_t sp; const char* name; } vs[] = {
      {0, 0, "poller echoes directly"}, {1, 0, "1 poller -> smem -> echo"}, {2, 300, "2 pollers (300 ns) -> smem"},
      {2, 500, "2 pollers (500 ns) -> smem"}};
  for (int trial = 0; trial < 2; ++trial)
    for (auto vv : vs) {
      memset(cells, 0, bytes);
      volatile unsigned long long* flags = cells;
      volatile unsigned long long* echo = cells + 2 * 16 * nsm + 512;
      k<<<nsm, 96, 0, st>>>((const unsigned long long*)flags, (unsigned long long*)echo, R, vv.mode, vv.sp);
      usleep(2000);
      std::vector<uint64_t> lat(R);
      bool bad = false;
      for (uint32_t r = 1; r <= R && !bad; ++r) {
        const uint32_t t = r % nsm;
        const uint64_t t0 = now_ns();
        if (r == R) {
          for (int i = 0; i < nsm; ++i) { flags[(i * 2) * 16] = R; flags[(i * 2 + 1) * 16] = R; }
        } else {
          flags[(t * 2) * 16] = r;
          flags[(t * 2 + 1) * 16] = r;
        }
        const uint64_t dl = t0 + 2000000000ull;
        while (echo[16 * t] != r) {
          _mm_pause();
          if (now_ns() > dl) { bad = true; break; }
        }
        lat[r - 1] = now_ns() - t0;
      }
      cudaStreamSynchronize(st);
      std::vector<uint64_t> s(lat.begin() + R / 10, lat.end() - 1);
      std::sort(s.begin(), s.end());
      auto q = [&](double p) { return s[size_t(p * (s.size() - 1))] / 1e3; };
      if (bad) printf("%s: stalled\n", vv.name);
      else printf("%-28s p10 %.3f p50 %.3f p90 %.3f p99.9 %.3f us\n", vv.name, q(0.1), q(0.5), q(0.9), q(0.999));
      fflush(stdout);
    }
  return 0;
}
