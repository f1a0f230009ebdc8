// probe_costs.cu -- device-side cost microbenchmarks for the LK hot path
// (design probe, not product code).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/probe_costs.cu -o tools/probe_costs
// Prints clock64 cycles for: a sys-scope store to pinned host memory (one, and
// two back to back to the same word), a gpu-scope store/load, %globaltimer
// reads, an L2 round trip, and the SM->SM latency of a store observed by a
// poller on another SM (the gateway's forwarding hop).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

__device__ __forceinline__ uint64_t clk() { uint64_t c; asm volatile("mov.u64 %0, %%clock64;" : "=l"(c)); return c; }
__device__ __forceinline__ uint64_t gtime() { uint64_t t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ void st_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_gpu(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_gpu(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__global__ void costs(unsigned long long* host, unsigned long long* dev, unsigned long long* out) {
  const int R = 64;
  uint64_t acc[8] = {0};
  for (int r = 0; r < R; ++r) {
    uint64_t c0 = clk(); st_sys(host, r); uint64_t c1 = clk(); acc[0] += c1 - c0;
    c0 = clk(); st_sys(host, r); st_sys(host, r + 1); c1 = clk(); acc[1] += c1 - c0;
    c0 = clk(); st_gpu(dev, r); c1 = clk(); acc[2] += c1 - c0;
    c0 = clk(); uint64_t t = gtime(); c1 = clk(); acc[3] += c1 - c0 + (t & 0);
    c0 = clk(); unsigned long long v = ld_gpu(dev + 64); c1 = clk(); acc[4] += c1 - c0 + (v & 0);
    c0 = clk(); st_sys(host + 16, r); unsigned long long w = ld_gpu(dev + 128); c1 = clk(); acc[5] += c1 - c0 + (w & 0);
    c0 = clk(); __threadfence_system(); c1 = clk(); acc[6] += c1 - c0;
    c0 = clk(); st_sys(host + 32, r); asm volatile("fence.acq_rel.sys;" ::: "memory"); c1 = clk(); acc[7] += c1 - c0;
  }
  for (int k = 0; k < 8; ++k) out[k] = acc[k] / R;
}

// block 0 writes seq r to `flag`, block 1 polls it and echoes; block 0 polls the echo.
__global__ void sm_hop(unsigned long long* flag, unsigned long long* echo, unsigned long long* out, int R) {
  if (threadIdx.x) return;
  if (blockIdx.x == 0) {
    uint64_t tot = 0, mx = 0;
    for (int r = 1; r <= R; ++r) {
      uint64_t c0 = clk();
      st_gpu(flag, r);
      while (ld_gpu(echo) != (unsigned long long)r) {}
      uint64_t d = clk() - c0;
      tot += d; mx = d > mx ? d : mx;
    }
    out[0] = tot / R; out[1] = mx;
  } else {
    for (int r = 1; r <= R; ++r) {
      while (ld_gpu(flag) != (unsigned long long)r) {}
      st_gpu(echo, r);
    }
  }
}

int main() {
  cudaSetDevice(0);
  unsigned long long *host, *dev, *out;
  cudaHostAlloc(&host, 4096, cudaHostAllocMapped);
  memset(host, 0, 4096);
  cudaMalloc(&dev, 65536);
  cudaMemset(dev, 0, 65536);
  cudaMallocManaged(&out, 4096);
  costs<<<1, 1>>>(host, dev, out);
  cudaDeviceSynchronize();
  const char* names[8] = {"st.relaxed.sys host (1)", "st.relaxed.sys host x2 same word", "st.relaxed.gpu dev",
                          "globaltimer read", "ld.relaxed.gpu L2 hit", "st.sys host + ld.gpu L2",
                          "__threadfence_system", "st.sys + fence.acq_rel.sys"};
  for (int k = 0; k < 8; ++k) printf("%-34s %6llu cycles\n", names[k], out[k]);
  cudaMemset(dev, 0, 65536);
  sm_hop<<<2, 32>>>(dev, dev + 4096, out, 10000);
  cudaDeviceSynchronize();
  printf("SM->SM L2 ping-pong (round trip)   avg %llu max %llu cycles\n", out[0], out[1]);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("clock rate attr %d kHz; err %s\n", clk_khz, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
