// probe_hot.cu -- 148 pollers; the host round-robins over the first 16
// ("hot") workers.  Do 2 staggered replica loads on the hot workers only
// shorten detection without the contention that made K=2 for everyone slower?
// (design probe, not product code)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_hot.cu -o tools/probe_hot
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
// worker i's K replica lines at flags[(i*2 + k) * 16]; hot workers (i < hot) poll k2 lines
__global__ void pollers(const unsigned long long* flags, unsigned long long* echo, uint32_t last, int hot, int k2,
                        uint32_t spacing) {
  if (threadIdx.x) return;
  const uint32_t i = blockIdx.x;
  const int K = int(i) < hot ? k2 : 1;
  const unsigned long long* f0 = flags + (i * 2) * 16;
  const unsigned long long* f1 = flags + (i * 2 + 1) * 16;
  unsigned long long* o = echo + 16 * i;
  unsigned long long seen = 0;
  unsigned long long v0 = ldr64(f0), v1 = 0;
  if (K == 2) { __nanosleep(spacing); v1 = ldr64(f1); }
  // consume the loads in issue order and reissue each at once, so the
  // replicas stay `spacing` apart
  for (;;) {
    if (v0 > seen) {
      seen = v0;
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(o), "l"(seen) : "memory");
      if (seen >= last) return;
    }
    v0 = ldr64(f0);
    if (K == 2) {
      if (v1 > seen) {
        seen = v1;
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(o), "l"(seen) : "memory");
        if (seen >= last) return;
      }
      v1 = ldr64(f1);
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
  const int hot = 16;
  struct V { int k2; uint32_t sp; } vs[] = {{1, 0}, {2, 0}, {2, 300}, {2, 500}};
  for (int trial = 0; trial < 2; ++trial)
    for (auto vv : vs) {
      memset(cells, 0, bytes);
      volatile unsigned long long* flags = cells;
      volatile unsigned long long* echo = cells + 2 * 16 * nsm + 512;
      pollers<<<nsm, 32, 0, st>>>((const unsigned long long*)flags, (unsigned long long*)echo, R, hot, vv.k2, vv.sp);
      usleep(2000);
      std::vector<uint64_t> lat(R);
      bool bad = false;
      for (uint32_t r = 1; r <= R && !bad; ++r) {
        const uint32_t t = r % hot;
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
      if (bad) printf("K=%d sp=%u stalled\n", vv.k2, vv.sp);
      else printf("hot 16 of %d, K=%d spacing %3u ns: p10 %.3f p50 %.3f p90 %.3f p99.9 %.3f us\n", nsm, vv.k2, vv.sp,
                  q(0.1), q(0.5), q(0.9), q(0.999));
      fflush(stdout);
    }
  return 0;
}
