// probe_shared.cu -- do 148 SMs polling ONE host line cost less per round trip
// than 148 SMs polling one line each?  (design probe, not product code)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_shared.cu -o tools/probe_shared
// A: per-SM lines (LK DIRECT today).  B: one shared line {round:24, target:8}.
// Round robin target = r % nsm; the target echoes r into its own echo line.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <time.h>
#include <unistd.h>
#include <immintrin.h>

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

__global__ void shared_line(const uint32_t* flag, uint32_t* echo, uint32_t last, uint32_t nsm) {
  if (threadIdx.x) return;
  uint32_t seen = 0;
  for (;;) {
    const uint32_t v = ldr(flag);
    if (v != seen) {
      seen = v;
      const uint32_t r = v >> 8, t = v & 0xFF;
      if (t == blockIdx.x) str(echo + 32 * blockIdx.x, r);
      if (r >= last) return;
    }
  }
}

static void report(const char* label, std::vector<uint64_t>& v) {
  std::vector<uint64_t> s(v.begin() + v.size() / 10, v.end());
  std::sort(s.begin(), s.end());
  auto q = [&](double p) { return s[std::min(s.size() - 1, size_t(p * s.size()))] / 1e3; };
  printf("%-40s p50 %6.3f  p99 %6.3f  p99.9 %6.3f us\n", label, q(0.5), q(0.99), q(0.999));
  fflush(stdout);
}

int main() {
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
  for (int grid : {nsm, 16}) {
    for (int mode = 0; mode < 2; ++mode) {
      memset(cells, 0, bytes);
      volatile uint32_t* flags = cells;                       // own lines: 32 u32 apart
      volatile uint32_t* echo = cells + 32 * nsm + 1024;      // own echo lines
      if (mode == 0) own_lines<<<grid, 32, 0, st>>>((const uint32_t*)flags, (uint32_t*)echo, R);
      else shared_line<<<grid, 32, 0, st>>>((const uint32_t*)flags, (uint32_t*)echo, R, grid);
      usleep(2000);
      std::vector<uint64_t> lat(R);
      bool bad = false;
      for (uint32_t r = 1; r <= R && !bad; ++r) {
        const uint32_t t = r % grid;
        const uint64_t t0 = now_ns();
        if (mode == 0) {
          if (r == R) for (int i = 0; i < grid; ++i) flags[32 * i] = R;   // release every poller
          else flags[32 * t] = r;
        } else {
          flags[0] = (r << 8) | t;
        }
        const uint64_t dl = t0 + 2000000000ull;
        while (echo[32 * t] != r) {
          _mm_pause();
          if (now_ns() > dl) { bad = true; break; }
        }
        lat[r - 1] = now_ns() - t0;
      }
      if (mode == 1) { flags[0] = (R << 8) | 0xFF; }
      cudaStreamSynchronize(st);
      char label[96];
      snprintf(label, sizeof label, "%s, %d SMs polling", mode ? "one shared line" : "own line per SM", grid);
      if (bad) printf("%s: stalled\n", label); else report(label, lat);
    }
  }
  return 0;
}
