// probe_link2.cu -- host->GPU mailbox write strategies (design probe, not product code).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -mclflushopt,-mcldemote tools/probe_link2.cu -o tools/probe_link2
// P pollers (one thread each, own 128-B line, one relaxed.sys load in flight) spin on
// host cells; the host pings poller (r % P) round robin, the poller echoes into its
// own echo line.  Variants: how the host writes the cell (plain store, + clflushopt,
// + cldemote, non-temporal store, write-combining mapping) and P.
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

__global__ void pollers(const uint32_t* cells, uint32_t* echo, uint32_t rounds_each) {
  const uint32_t* c = cells + 32 * blockIdx.x;
  uint32_t* e = echo + 32 * blockIdx.x;
  for (uint32_t r = 1; r <= rounds_each; ++r) {
    uint32_t v;
    do {
      asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
    } while (v != r);
    asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(e), "r"(r) : "memory");
  }
}

enum Mode { PLAIN, FLUSH, DEMOTE, NT, WC };
static const char* names[] = {"plain store", "store+clflushopt", "store+cldemote", "movnti", "WC mapping"};

static void run(int P, Mode m, int rounds_each, bool has_demote) {
  if (m == DEMOTE && !has_demote) { printf("P=%3d %-18s (no cldemote)\n", P, names[m]); return; }
  uint32_t *cells, *echo;
  cudaHostAlloc(&cells, size_t(P) * 128, cudaHostAllocMapped | (m == WC ? cudaHostAllocWriteCombined : 0));
  cudaHostAlloc(&echo, size_t(P) * 128, cudaHostAllocMapped);
  memset(echo, 0, size_t(P) * 128);
  for (int i = 0; i < P; ++i) cells[32 * i] = 0;
  _mm_sfence();
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  pollers<<<P, 1, 0, st>>>(cells, echo, rounds_each);
  usleep(2000);
  std::vector<uint64_t> lat;
  const int R = P * rounds_each;
  lat.reserve(R);
  bool stalled = false;
  for (int k = 0; k < R && !stalled; ++k) {
    const int i = k % P;
    const uint32_t want = uint32_t(k / P + 1);
    uint32_t* c = cells + 32 * i;
    volatile uint32_t* e = echo + 32 * i;
    const uint64_t t0 = now_ns();
    switch (m) {
      case PLAIN: *(volatile uint32_t*)c = want; break;
      case FLUSH: *(volatile uint32_t*)c = want; _mm_clflushopt(c); break;
#ifdef __CLDEMOTE__
      case DEMOTE: *(volatile uint32_t*)c = want; _cldemote(c); break;
#else
      case DEMOTE: break;
#endif
      case NT: _mm_stream_si32(reinterpret_cast<int*>(c), int(want)); _mm_sfence(); break;
      case WC: *(volatile uint32_t*)c = want; _mm_sfence(); break;
    }
    const uint64_t dl = t0 + 1000000000ull;
    while (*e != want) {
      _mm_pause();
      if (now_ns() > dl) { stalled = true; break; }
    }
    if (k >= P) lat.push_back(now_ns() - t0);
  }
  cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  cudaFreeHost(cells);
  cudaFreeHost(echo);
  if (stalled) { printf("P=%3d %-18s stalled\n", P, names[m]); return; }
  std::sort(lat.begin(), lat.end());
  auto q = [&](double p) { return lat[std::min(lat.size() - 1, size_t(p * lat.size()))] / 1e3; };
  printf("P=%3d %-18s p50 %6.3f p90 %6.3f p99 %6.3f p99.9 %6.3f us\n", P, names[m], q(.5), q(.9), q(.99), q(.999));
  fflush(stdout);
}

int main() {
  cudaSetDevice(0);
  cudaFree(0);
  bool has_demote = __builtin_cpu_supports("cldemote");
  printf("cpu cldemote=%d\n", int(has_demote));
  for (int P : {1, 4, 16, 64, 148}) {
    for (int m = PLAIN; m <= WC; ++m) run(P, Mode(m), std::max(20000 / P, 100), has_demote);
  }
  return 0;
}
