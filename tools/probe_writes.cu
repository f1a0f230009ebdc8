// probe_writes.cu -- does the SIZE of the device's echo store change the
// host<->GPU ping-pong?  Partial-line DMA writes may need a read-for-ownership
// at the host; full 64-B lines may not.  (design probe, not product code)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_writes.cu -o tools/probe_writes
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
__device__ __forceinline__ uint64_t ldr64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// mode 0: lane 0 stores 8 B; 1: lane 0 stores 16 B (v2.u64); 2: lanes 0-3 store 32 B;
// 3: lanes 0-7 store 64 B (one full line); 4: lanes 0-15 store 128 B; 5: lane 0 stores 32 B
// with one 256-bit store (sm_100)
__global__ void echo(const unsigned long long* flag, unsigned long long* out, uint32_t rounds, int mode) {
  const uint32_t lane = threadIdx.x;
  unsigned long long seen = 0;
  for (uint32_t r = 1; r <= rounds; ++r) {
    unsigned long long v = 0;
    if (lane == 0) {
      do { v = ldr64(flag); } while (v == seen);
    }
    v = __shfl_sync(0xffffffffu, v, 0);
    seen = v;
    if (mode == 0) {
      if (lane == 0) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(out), "l"(v) : "memory");
    } else if (mode == 6) {   // 2 lanes x 16 B
      if (lane < 2) asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %1};" ::"l"(out + 2 * lane), "l"(v) : "memory");
    } else if (mode == 7) {   // 4 lanes x 8 B, lanes 1-3 on other lines
      if (lane < 4) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(out + 16 * lane), "l"(v) : "memory");
    } else if (mode == 8) {   // 4 lanes, same 8 B
      if (lane < 4) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(out), "l"(v) : "memory");
    } else if (mode == 9) {   // 2 lanes x 8 B (16 B)
      if (lane < 2) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(out + lane), "l"(v) : "memory");
    } else if (mode == 10) {  // 2 lanes, same 8 B
      if (lane < 2) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(out), "l"(v) : "memory");
    } else if (mode == 11) {  // 32 lanes, same 8 B
      asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(out), "l"(v) : "memory");
    } else if (mode == 12) {  // lane 0 stores the same 8 B twice
      if (lane == 0) {
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(out), "l"(v) : "memory");
        asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(out), "l"(v) : "memory");
      }
    } else if (mode == 5) {
      if (lane == 0) asm volatile("st.relaxed.sys.global.v4.u64 [%0], {%1, %1, %1, %1};" ::"l"(out), "l"(v) : "memory");
    } else if (mode == 1) {
      if (lane == 0) asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %1};" ::"l"(out), "l"(v) : "memory");
    } else {
      const uint32_t n = mode == 2 ? 4 : mode == 3 ? 8 : 16;
      if (lane < n) asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(out + lane), "l"(v) : "memory");
    }
  }
}

int main() {
  cudaSetDevice(0);
  cudaFree(0);
  unsigned long long* cells;
  cudaHostAlloc(&cells, 8192, cudaHostAllocMapped | cudaHostAllocPortable);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  const uint32_t R = 30000;
  const char* names[] = {"8 B, 1 lane", "16 B, 1 lane (v2)", "32 B, 4 lanes", "64 B, 8 lanes (full line)",
                         "128 B, 16 lanes", "32 B, 1 lane (256-bit store)",
                         "32 B, 2 lanes x v2", "4 lanes, 4 lines", "4 lanes, same 8 B", "16 B, 2 lanes",
                         "2 lanes, same 8 B", "32 lanes, same 8 B", "1 lane, same 8 B twice"};
  for (int trial = 0; trial < 2; ++trial)
    for (int mode : {0, 8, 10, 11, 12, 2, 9}) {
      memset(cells, 0, 8192);
      volatile unsigned long long* flag = cells;
      volatile unsigned long long* out = cells + 512;   // 4 KiB away, 128-B aligned
      echo<<<1, 32, 0, st>>>((const unsigned long long*)flag, (unsigned long long*)out, R, mode);
      usleep(2000);
      std::vector<uint64_t> lat(R);
      bool bad = false;
      for (uint32_t r = 1; r <= R && !bad; ++r) {
        const uint64_t t0 = now_ns();
        *flag = r;
        const uint64_t dl = t0 + 2000000000ull;
        while (out[0] != r) {
          _mm_pause();
          if (now_ns() > dl) { bad = true; break; }
        }
        lat[r - 1] = now_ns() - t0;
      }
      cudaStreamSynchronize(st);
      std::vector<uint64_t> s(lat.begin() + R / 10, lat.end());
      std::sort(s.begin(), s.end());
      if (bad) printf("%-28s stalled\n", names[mode]);
      else {
        auto q = [&](double p) { return s[size_t(p * (s.size() - 1))] / 1e3; };
        printf("%-28s p10 %6.3f p25 %6.3f p50 %6.3f p75 %6.3f p90 %6.3f p99 %6.3f us\n", names[mode], q(0.1),
               q(0.25), q(0.5), q(0.75), q(0.9), q(0.99));
      }
      fflush(stdout);
    }
  return 0;
}
