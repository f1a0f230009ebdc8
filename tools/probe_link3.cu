// probe_link3.cu -- P pollers x K staggered replica loads (design probe, not product code).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_link3.cu -o tools/probe_link3
// Each poller (one thread per block) owns a cell with K replica lines; one load
// in flight per replica, staggered d ns.  The host pings poller (r % P) round
// robin (writing all K replicas) and waits for the echo.  Question: does
// (P/2 pollers, 2K loads each) beat (P pollers, K loads) at equal in-flight count?
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
__device__ __forceinline__ uint32_t ldr(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

template <int K>
__global__ void pollers(const uint32_t* cells, uint32_t* echo, uint32_t rounds_each, uint32_t d) {
  const uint32_t* c = cells + 32 * K * blockIdx.x;   // replica k at c + 32k
  uint32_t* e = echo + 32 * blockIdx.x;
  for (uint32_t r = 1; r <= rounds_each; ++r) {
    uint32_t v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) { v[k] = ldr(c + 32 * k); if (K > 1) __nanosleep(d); }
    bool done = false;
    while (!done) {
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if (v[k] == r) { done = true; break; }
        v[k] = ldr(c + 32 * k);
        if (K > 1) __nanosleep(d);
      }
    }
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(e), "r"(r) : "memory");
  }
}

static void run(int P, int K, uint32_t d) {
  const int rounds_each = std::max(30000 / P, 50);
  uint32_t *cells, *echo;
  cudaHostAlloc(&cells, size_t(P) * K * 128, cudaHostAllocMapped);
  cudaHostAlloc(&echo, size_t(P) * 128, cudaHostAllocMapped);
  memset(cells, 0, size_t(P) * K * 128);
  memset(echo, 0, size_t(P) * 128);
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  switch (K) {
    case 1: pollers<1><<<P, 1, 0, st>>>(cells, echo, rounds_each, d); break;
    case 2: pollers<2><<<P, 1, 0, st>>>(cells, echo, rounds_each, d); break;
    case 4: pollers<4><<<P, 1, 0, st>>>(cells, echo, rounds_each, d); break;
  }
  usleep(2000);
  std::vector<uint64_t> lat;
  bool stalled = false;
  for (int k = 0; k < P * rounds_each && !stalled; ++k) {
    const int i = k % P;
    const uint32_t want = uint32_t(k / P + 1);
    volatile uint32_t* e = echo + 32 * i;
    const uint64_t t0 = now_ns();
    for (int q = K - 1; q >= 0; --q) *(volatile uint32_t*)(cells + 32 * (K * i + q)) = want;
    const uint64_t dl = t0 + 1000000000ull;
    while (*e != want) { _mm_pause(); if (now_ns() > dl) { stalled = true; break; } }
    if (k >= P) lat.push_back(now_ns() - t0);
  }
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  cudaFreeHost(cells);
  cudaFreeHost(echo);
  if (stalled) { printf("P=%3d K=%d d=%4u stalled\n", P, K, d); return; }
  std::sort(lat.begin(), lat.end());
  auto q = [&](double p) { return lat[std::min(lat.size() - 1, size_t(p * lat.size()))] / 1e3; };
  printf("P=%3d K=%d d=%4u in-flight=%3d  p50 %6.3f p90 %6.3f p99 %6.3f p99.9 %6.3f us\n", P, K, d, P * K, q(.5),
         q(.9), q(.99), q(.999));
  fflush(stdout);
}

int main() {
  cudaSetDevice(0);
  cudaFree(0);
  run(148, 1, 0);
  run(74, 2, 400); run(74, 2, 800);
  run(37, 4, 200); run(37, 4, 400);
  run(148, 2, 400); run(148, 2, 800);
  run(74, 1, 0);
  run(37, 2, 400);
  run(16, 2, 400); run(16, 4, 300);
  run(1, 2, 400); run(1, 2, 800);
  return 0;
}
