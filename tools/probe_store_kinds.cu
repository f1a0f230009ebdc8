// probe_store_kinds.cu -- which device store makes a value visible to a host
// poller soonest?  148 SMs, one polled line each, round robin (LK DIRECT
// shape); only the echo store differs.  (design probe, not product code)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_store_kinds.cu -o tools/probe_store_kinds
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
template <int M>
__device__ __forceinline__ void store(unsigned long long* o, unsigned long long v) {
  if (M == 0) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(o), "l"(v) : "memory");
  if (M == 1) asm volatile("st.global.wt.u64 [%0], %1;" ::"l"(o), "l"(v) : "memory");
  if (M == 2) asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(o), "l"(v) : "memory");
  if (M == 3) asm volatile("st.global.cg.u64 [%0], %1;" ::"l"(o), "l"(v) : "memory");
  if (M == 4) asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(o), "l"(v) : "memory");
  if (M == 5) asm volatile("st.relaxed.sys.global.u64 [%0], %1; fence.sc.sys;" ::"l"(o), "l"(v) : "memory");
  if (M == 6) {
    unsigned long long old;
    asm volatile("atom.relaxed.sys.global.exch.b64 %0, [%1], %2;" : "=l"(old) : "l"(o), "l"(v) : "memory");
  }
  if (M == 7) asm volatile("st.relaxed.sys.global.u64 [%0], %1; fence.proxy.alias;" ::"l"(o), "l"(v) : "memory");
}
template <int M>
__global__ void own_lines(const unsigned long long* flags, unsigned long long* echo, uint32_t last) {
  if (threadIdx.x) return;
  const unsigned long long* f = flags + 16 * blockIdx.x;
  unsigned long long* o = echo + 16 * blockIdx.x;
  unsigned long long seen = 0;
  for (;;) {
    const unsigned long long v = ldr64(f);
    if (v != seen) {
      seen = v;
      store<M>(o, v);
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
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const char* names[] = {"st.relaxed.sys (LK today)", "st.global.wt", "st.volatile", "st.global.cg", "st.release.sys",
                         "st.relaxed.sys + fence.sc.sys", "atom.exch.relaxed.sys", "st.relaxed.sys + fence.proxy"};
  for (int trial = 0; trial < 2; ++trial)
    for (int m = 0; m < 8; ++m) {
      memset(cells, 0, bytes);
      volatile unsigned long long* flags = cells;
      volatile unsigned long long* echo = cells + 16 * nsm + 512;
      const unsigned long long* fp = (const unsigned long long*)flags;
      unsigned long long* ep = (unsigned long long*)echo;
      switch (m) {
        case 0: own_lines<0><<<nsm, 32, 0, st>>>(fp, ep, R); break;
        case 1: own_lines<1><<<nsm, 32, 0, st>>>(fp, ep, R); break;
        case 2: own_lines<2><<<nsm, 32, 0, st>>>(fp, ep, R); break;
        case 3: own_lines<3><<<nsm, 32, 0, st>>>(fp, ep, R); break;
        case 4: own_lines<4><<<nsm, 32, 0, st>>>(fp, ep, R); break;
        case 5: own_lines<5><<<nsm, 32, 0, st>>>(fp, ep, R); break;
        case 6: own_lines<6><<<nsm, 32, 0, st>>>(fp, ep, R); break;
        case 7: own_lines<7><<<nsm, 32, 0, st>>>(fp, ep, R); break;
      }
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
      if (bad) printf("%-32s stalled\n", names[m]);
      else printf("%-32s p10 %.3f p50 %.3f p90 %.3f p99.9 %.3f us\n", names[m], q(0.1), q(0.5), q(0.9), q(0.999));
      fflush(stdout);
    }
  return 0;
}
