// probe_rr_store.cu -- 148 SMs, one polled line each (LK DIRECT shape), round
// robin: echo with a 1-lane store vs the same 8 B stored by 2 lanes of the
// warp (tools/probe_writes.cu found the latter ~1 us faster for one poller).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_rr_store.cu -o tools/probe_rr_store
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
// lanes [0, nl) poll (one coalesced load) and store the echo
__global__ void own_lines(const unsigned long long* flags, unsigned long long* echo, uint32_t last, int nl) {
  const uint32_t lane = threadIdx.x;
  if (lane >= uint32_t(nl)) return;
  const unsigned long long* f = flags + 16 * blockIdx.x;
  unsigned long long* o = echo + 16 * blockIdx.x;
  unsigned long long seen = 0;
  for (;;) {
    const unsigned long long v = ldr64(f);
    if (v != seen) {
      seen = v;
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(o), "l"(v) : "memory");
      if (v >= last) return;
    }
  }
}

int main() {
  cudaSetDevice(0);
  cudaFree(0);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const uint32_t R = 60000;
  unsigned long long* cells;
  const size_t bytes = size_t(nsm) * 128 * 2 + 4096;
  cudaHostAlloc(&cells, bytes, cudaHostAllocMapped | cudaHostAllocPortable);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int trial = 0; trial < 2; ++trial)
    for (int nl : {1, 2, 4, 32}) {
      memset(cells, 0, bytes);
      volatile unsigned long long* flags = cells;
      volatile unsigned long long* echo = cells + 16 * nsm + 512;
      own_lines<<<nsm, 32, 0, st>>>((const unsigned long long*)flags, (unsigned long long*)echo, R, nl);
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
      if (bad) printf("%d lanes: stalled\n", nl);
      else printf("%2d lane(s) poll+store: p10 %.3f p50 %.3f p90 %.3f p99 %.3f p99.9 %.3f us\n", nl, q(0.1), q(0.5),
                  q(0.9), q(0.99), q(0.999));
      fflush(stdout);
    }
  return 0;
}
