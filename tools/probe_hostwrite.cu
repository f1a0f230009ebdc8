// probe_hostwrite.cu -- does HOW the host writes a mailbox word change the
// host->GPU->host round trip?  (design probe, not product code)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -mclflushopt,-mcldemote,-mclwb
//        tools/probe_hostwrite.cu -o tools/probe_hostwrite
// 148 SMs, one line each (LK DIRECT); round robin; the target echoes into
// its own status line.  Variants of the host store: plain mov, + clflushopt,
// + clwb, + cldemote, non-temporal movnti + sfence.
#include <cuda_runtime.h>
#include <immintrin.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <time.h>
#include <unistd.h>
#include <cpuid.h>

#include <algorithm>
#include <vector>

static inline uint64_t now_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return uint64_t(ts.tv_sec) * 1000000000ull + ts.tv_nsec;
}
__device__ __forceinline__ uint32_t ldr(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void str(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__global__ void own_lines(const uint32_t* flags, uint32_t* echo, uint32_t last) {
  if (threadIdx.x) return;
  const uint32_t* f = flags + 32 * blockIdx.x;
  uint32_t seen = 0;
  for (;;) {
    const uint32_t v = ldr(f);
    if (v != seen) {
      seen = v;
      str(echo + 32 * blockIdx.x, v);
      if (v >= last) return;
    }
  }
}

static void report(const char* label, std::vector<uint64_t>& v) {
  std::vector<uint64_t> s(v.begin() + v.size() / 10, v.end());
  std::sort(s.begin(), s.end());
  auto q = [&](double p) { return s[std::min(s.size() - 1, size_t(p * s.size()))] / 1e3; };
  printf("%-28s p50 %6.3f  p99 %6.3f  p99.9 %6.3f us\n", label, q(0.5), q(0.99), q(0.999));
  fflush(stdout);
}

__attribute__((target("clflushopt,clwb,cldemote"))) static inline void do_write(int how, volatile uint32_t* p,
                                                                               uint32_t v) {
  switch (how) {
    case 0: *p = v; break;
    case 1: *p = v; _mm_clflushopt((void*)p); break;
    case 2: *p = v; _mm_clwb((void*)p); break;
    case 3: *p = v; _cldemote((void*)p); break;
    case 4: _mm_stream_si32((int*)p, int(v)); _mm_sfence(); break;
    case 5: *p = v; _mm_sfence(); break;
  }
}

int main() {
  unsigned a, b, c, d;
  __cpuid_count(7, 0, a, b, c, d);
  const bool has_clflushopt = b & (1u << 23), has_clwb = b & (1u << 24), has_cldemote = c & (1u << 25);
  printf("cpu: clflushopt %d clwb %d cldemote %d\n", has_clflushopt, has_clwb, has_cldemote);
  cudaSetDevice(0);
  cudaFree(0);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const uint32_t R = 40000;
  uint32_t* cells;
  const size_t bytes = size_t(nsm) * 128 * 2 + 4096;
  cudaHostAlloc(&cells, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const char* names[] = {"plain store", "store+clflushopt", "store+clwb", "store+cldemote", "movnti+sfence",
                         "store+sfence"};
  for (int trial = 0; trial < 2; ++trial)
    for (int how = 0; how < 6; ++how) {
      if ((how == 1 && !has_clflushopt) || (how == 2 && !has_clwb) || (how == 3 && !has_cldemote)) continue;
      memset(cells, 0, bytes);
      volatile uint32_t* flags = cells;
      volatile uint32_t* echo = cells + 32 * nsm + 1024;
      own_lines<<<nsm, 32, 0, st>>>((const uint32_t*)flags, (uint32_t*)echo, R);
      usleep(2000);
      std::vector<uint64_t> lat(R);
      bool bad = false;
      for (uint32_t r = 1; r <= R && !bad; ++r) {
        const uint32_t t = r % nsm;
        const uint64_t t0 = now_ns();
        if (r == R) for (int i = 0; i < nsm; ++i) flags[32 * i] = R;
        else do_write(how, flags + 32 * t, r);
        const uint64_t dl = t0 + 2000000000ull;
        while (echo[32 * t] != r) {
          _mm_pause();
          if (now_ns() > dl) { bad = true; break; }
        }
        lat[r - 1] = now_ns() - t0;
      }
      cudaStreamSynchronize(st);
      if (bad) printf("%s: stalled\n", names[how]); else report(names[how], lat);
    }
  return 0;
}
