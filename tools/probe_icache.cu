// Does an acquire (CCTL.IVALL) or a sys-scope fence evict the instruction
// cache?  One thread times a 2 KB noinline function cold, warm, and warm
// again after each candidate operation.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/probe_icache tools/probe_icache.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __noinline__ uint32_t body(uint32_t x) {
#pragma unroll
  for (int i = 0; i < 128; ++i) x = (x ^ (x >> 7)) * 1664525u + uint32_t(i);
  return x;
}

template <int N>
__device__ __noinline__ uint32_t evict(uint32_t x) {
#pragma unroll
  for (int i = 0; i < N; ++i) x = (x ^ (x >> 5)) * 22695477u + uint32_t(i);
  return x;
}

__device__ __forceinline__ uint64_t clk() { uint64_t c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c; }
// a clock read that waits for r, and an r that waits for the clock read
__device__ __forceinline__ uint64_t clk_after(uint32_t r) {
  uint64_t c;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(c) : "r"(r) : "memory");
  return c;
}
__device__ __forceinline__ uint32_t tie(uint32_t r, uint64_t t) {
  asm volatile("" : "+r"(r) : "l"(t));
  return r;
}

__global__ void probe(uint64_t* out, uint32_t* g, int mode) {
  if (threadIdx.x) return;
  uint32_t r = 1;
  const uint64_t t0 = clk_after(r); r = body(tie(r, t0)); const uint64_t t1 = clk_after(r);
  r = body(tie(r, t1)); const uint64_t t2 = clk_after(r);
  volatile uint32_t loc[8];
  const uint32_t li = g[1] & 7;   // a run-time index keeps loc in local memory
  loc[li] = r;
  uint32_t v = 0;
  switch (mode) {
    case 1: asm volatile("fence.acq_rel.gpu;" ::: "memory"); break;
    case 2: asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(g) : "memory"); break;
    case 3: asm volatile("fence.acq_rel.sys;" ::: "memory"); break;
    case 4: asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(g) : "memory"); break;
    case 5: { const uint64_t e = clk() + 20000; while (clk() < e) {} } break;   // ~10 us of a tight loop
    case 6: asm volatile("fence.proxy.async.global;" ::: "memory"); break;
    case 7: asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(g) : "memory"); break;
    case 8: v = evict<170>(r) == 0x9e3779b9u; break;     // ~8 KB of other code
    case 9: v = evict<340>(r) == 0x9e3779b9u; break;     // ~16 KB
    case 10: v = evict<510>(r) == 0x9e3779b9u; break;    // ~24 KB
    case 11: v = evict<680>(r) == 0x9e3779b9u; break;    // ~32 KB
    case 12: v = evict<1020>(r) == 0x9e3779b9u; break;   // ~48 KB
    case 13: v = evict<1360>(r) == 0x9e3779b9u; break;   // ~64 KB
    default: break;
  }
  r += v;
  const uint64_t t5 = clk_after(r);
  const uint32_t y = loc[li ^ (tie(r, t5) & 0)];           // a local-memory (spill-like) load after the op
  const uint64_t t6 = clk_after(y);
  r += y;
  const uint64_t t3 = clk_after(r); r = body(tie(r, t3)); const uint64_t t4 = clk_after(r);
  out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t4 - t3; out[3] = r; out[4] = t6 - t5;
}

int main() {
  uint64_t* d; uint32_t* g; cudaMalloc(&d, 128); cudaMalloc(&g, 64); cudaMemset(g, 0, 64);
  const char* names[] = {"nothing", "fence.acq_rel.gpu", "ld.acquire.gpu", "fence.acq_rel.sys", "ld.acquire.sys",
                         "10 us spin", "fence.proxy.async", "ld.relaxed.sys", "8 KB other code",
                         "16 KB other code", "24 KB other code", "32 KB other code", "48 KB other code",
                         "64 KB other code"};
  for (int mode = 0; mode < 14; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      probe<<<1, 32>>>(d, g, mode);
      uint64_t h[5];
      cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
      printf("%-20s rep %d: cold %5llu  warm %5llu  after op %5llu cycles | local load after op %4llu\n", names[mode],
             rep, (unsigned long long)h[0], (unsigned long long)h[1], (unsigned long long)h[2],
             (unsigned long long)h[4]);
    }
  }
  return 0;
}
