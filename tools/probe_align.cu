// probe_align.cu -- closed-loop round robin over 148 pollers: after any SM
// publishes an echo (which the host answers with the next write, to another
// SM), do polls aligned to "last publish + D" find the host's write sooner
// than free-running polls?  (design probe, not product code)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_align.cu -o tools/probe_align
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
__device__ __forceinline__ unsigned long long ldgpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// D == 0: free-running polls.  Else: before each load, wait until
// last_pub + D if that is in the future.
__global__ void pollers(const unsigned long long* flags, unsigned long long* echo, unsigned long long* last_pub,
                        uint32_t last, uint32_t D) {
  if (threadIdx.x) return;
  const unsigned long long* f = flags + 16 * blockIdx.x;
  unsigned long long* o = echo + 16 * blockIdx.x;
  unsigned long long seen = 0;
  for (;;) {
    if (D >= 10000) {   // pure throttle: a gap of D - 10000 ns before each host load
      const unsigned long long t = gtime() + (D - 10000);
      while (gtime() < t) {
      }
    } else if (D) {   // D == 1: the L2 read only (its cost), no wait
      const unsigned long long t = ldgpu(last_pub) + (D > 1 ? D : 0);
      while (D > 1 && gtime() < t) {
      }
    }
    const unsigned long long v = ldr64(f);
    if (v != seen) {
      seen = v;
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(o), "l"(v) : "memory");
      if (D) asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(last_pub), "l"(gtime()) : "memory");
      if (v >= last) return;
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
  const size_t bytes = size_t(nsm) * 128 * 2 + 4096;
  cudaHostAlloc(&cells, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
  unsigned long long* d_last;
  cudaMalloc(&d_last, 128);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int trial = 0; trial < 2; ++trial)
    for (uint32_t D : {0u, 1u, 10100u, 10200u, 10300u, 10500u, 10800u, 350u}) {
      memset(cells, 0, bytes);
      cudaMemset(d_last, 0, 128);
      cudaDeviceSynchronize();
      volatile unsigned long long* flags = cells;
      volatile unsigned long long* echo = cells + 16 * nsm + 512;
      pollers<<<nsm, 32, 0, st>>>((const unsigned long long*)flags, (unsigned long long*)echo, d_last, R, D);
      usleep(2000);
      std::vector<uint64_t> lat(R);
      bool bad = false;
      for (uint32_t r = 1; r <= R && !bad; ++r) {
        const uint32_t t = r % nsm;
        const uint64_t t0 = now_ns();
        if (r == R) for (int i = 0; i < nsm; ++i) flags[16 * i] = R;
        else flags[16 * t] = r;
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
      if (bad) printf("D=%u: stalled\n", D);
      else printf("align D=%4u ns: p10 %.3f p50 %.3f p90 %.3f p99.9 %.3f us\n", D, q(0.1), q(0.5), q(0.9), q(0.999));
      fflush(stdout);
    }
  return 0;
}
