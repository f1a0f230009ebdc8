// probe_hot2.cu -- like probe_hot.cu, but the hot workers' two replica lines
// are polled by two different warps of the CTA (one load in flight each,
// started `spacing` apart); the first warp to see the new value echoes it.
// Does a second polling warp halve the detection residual?  (design probe)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_hot2.cu -o tools/probe_hot2
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
__global__ void pollers(const unsigned long long* flags, unsigned long long* echo, uint32_t last, int hot, int nw,
                        uint32_t spacing) {
  __shared__ unsigned long long best;
  if (threadIdx.x == 0) best = 0;
  __syncthreads();
  const uint32_t i = blockIdx.x, w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) != 0) return;
  const int W = int(i) < hot ? nw : 1;
  if (int(w) >= W) return;
  const unsigned long long* f = flags + (i * 2 + w) * 16;
  unsigned long long* o = echo + 16 * i;
  if (w) __nanosleep(spacing);
  for (;;) {
    const unsigned long long v = ldr64(f);
    if (v > *(volatile unsigned long long*)&best) {
      if (atomicMax(&best, v) < v) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(o), "l"(v) : "memory");
      if (v >= last) return;
    }
    if (*(volatile unsigned long long*)&best >= last) return;
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
  struct V { int hot, nw; uint32_t sp; } vs[] = {{16, 1, 0}, {16, 2, 300}, {16, 2, 500}, {148, 1, 0}, {148, 2, 500}};
  for (int trial = 0; trial < 2; ++trial)
    for (auto vv : vs) {
      memset(cells, 0, bytes);
      volatile unsigned long long* flags = cells;
      volatile unsigned long long* echo = cells + 2 * 16 * nsm + 512;
      pollers<<<nsm, 64, 0, st>>>((const unsigned long long*)flags, (unsigned long long*)echo, R, vv.hot, vv.nw, vv.sp);
      usleep(2000);
      std::vector<uint64_t> lat(R);
      bool bad = false;
      for (uint32_t r = 1; r <= R && !bad; ++r) {
        const uint32_t t = r % vv.hot;
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
      if (bad) printf("stalled\n");
      else printf("round robin over %3d of %d, %d polling warp(s) each, spacing %3u ns: p10 %.3f p50 %.3f p90 %.3f "
                  "p99.9 %.3f us\n", vv.hot, nsm, vv.nw, vv.sp, q(0.1), q(0.5), q(0.9), q(0.999));
      fflush(stdout);
    }
  return 0;
}
