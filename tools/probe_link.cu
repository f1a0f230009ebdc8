// probe_link.cu -- host<->GPU word round-trip microbenchmarks (design probe,
// not product code).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   tools/probe_link.cu -o tools/probe_link -lcuda
//
//  A. single poller ping-pong over pinned mapped host memory
//  B. K staggered polls in flight (spacing d ns) -- lower detection latency?
//  C. host writes into DEVICE memory through a dma-buf BAR1 mmap (if the
//     driver allows CPU mmap of the exported range), GPU polls its own L2
#include <cuda.h>
#include <cuda_runtime.h>
#include <errno.h>
#include <fcntl.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
#include <sys/mman.h>
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
__device__ __forceinline__ uint32_t ldv(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void str(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int K>
__global__ void pp_staggered(const uint32_t* flag, uint32_t* echo, uint64_t rounds, uint32_t d) {
  for (uint64_t r = 1; r <= rounds; ++r) {
    const uint32_t want = uint32_t(r);
    uint32_t v[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      v[i] = ldr(flag);
      if (K > 1) __nanosleep(d);
    }
    bool done = false;
    while (!done) {
#pragma unroll
      for (int i = 0; i < K; ++i) {
        if (v[i] == want) { done = true; break; }
        v[i] = ldr(flag);
        if (K > 1) __nanosleep(d);
      }
    }
    str(echo, want);
  }
}

// K replica flags (128 B apart), one load in flight per replica, staggered.
template <int K>
__global__ void pp_replica(const uint32_t* flag, uint32_t* echo, uint64_t rounds, uint32_t d) {
  for (uint64_t r = 1; r <= rounds; ++r) {
    const uint32_t want = uint32_t(r);
    uint32_t v[K];
#pragma unroll
    for (int i = 0; i < K; ++i) { v[i] = ldr(flag + 32 * i); __nanosleep(d); }
    bool done = false;
    while (!done) {
#pragma unroll
      for (int i = 0; i < K; ++i) {
        if (v[i] == want) { done = true; break; }
        v[i] = ldr(flag + 32 * i);
        __nanosleep(d);
      }
    }
    str(echo, want);
  }
}

// W warps poll the same word, staggered by d; the first to see it echoes.
__global__ void pp_warps(const uint32_t* flag, uint32_t* echo, uint64_t rounds, uint32_t d) {
  __shared__ volatile uint32_t seen;
  const uint32_t w = threadIdx.x >> 5;
  if (threadIdx.x == 0) seen = 0;
  __syncthreads();
  for (uint64_t r = 1; r <= rounds; ++r) {
    const uint32_t want = uint32_t(r);
    if ((threadIdx.x & 31) == 0) {
      __nanosleep(w * d);
      for (;;) {
        if (seen >= want) break;
        const uint32_t v = ldr(flag);
        if (v == want) {
          if (atomicMax((uint32_t*)&seen, want) < want) str(echo, want);
          break;
        }
      }
    }
    __syncthreads();
  }
}

// Poll device memory written by the CPU through BAR1.
__global__ void pp_devflag(const uint32_t* dflag, uint32_t* echo, uint64_t rounds, int mode) {
  for (uint64_t r = 1; r <= rounds; ++r) {
    const uint32_t want = uint32_t(r);
    if (mode == 0) while (ldr(dflag) != want) {}
    else while (ldv(dflag) != want) {}
    str(echo, want);
  }
}

static void report(const char* label, std::vector<uint64_t>& v) {
  std::vector<uint64_t> s(v.begin() + std::min<size_t>(100, v.size() / 10), v.end());
  std::sort(s.begin(), s.end());
  auto q = [&](double p) { return s[std::min(s.size() - 1, size_t(p * s.size()))] / 1e3; };
  printf("%-34s p50 %6.3f  p99 %6.3f  p99.9 %6.3f  max %7.3f us\n", label, q(0.5), q(0.99), q(0.999),
         s.back() / 1e3);
  fflush(stdout);
}

static int host_loop(volatile uint32_t* flag, volatile uint32_t* echo, uint64_t rounds, std::vector<uint64_t>& out,
                     bool wc) {
  out.resize(rounds);
  for (uint64_t r = 1; r <= rounds; ++r) {
    const uint64_t t0 = now_ns();
    *flag = uint32_t(r);
    if (wc) _mm_sfence();
    const uint64_t dl = t0 + 2000000000ull;
    while (*echo != uint32_t(r)) {
      _mm_pause();
      if (now_ns() > dl) { printf("  stalled at round %llu\n", (unsigned long long)r); return -1; }
    }
    out[r - 1] = now_ns() - t0;
  }
  return 0;
}

int main() {
  cudaSetDevice(0);
  cudaFree(0);
  const uint64_t R = 20000;
  uint32_t* cells;
  cudaHostAlloc(&cells, 4096, cudaHostAllocMapped | cudaHostAllocPortable);
  memset(cells, 0, 4096);
  volatile uint32_t* flag = cells;
  volatile uint32_t* echo = cells + 32;
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  std::vector<uint64_t> lat;

  // A/B: staggered polling over host memory
  struct Cfg { int k; uint32_t d; } cfgs[] = {{1, 0}, {2, 300}, {2, 600}, {4, 150}, {4, 300}, {8, 100}, {8, 200}};
  for (auto c : cfgs) {
    memset(cells, 0, 4096);
    switch (c.k) {
      case 1: pp_staggered<1><<<1, 1, 0, st>>>((const uint32_t*)flag, (uint32_t*)echo, R, c.d); break;
      case 2: pp_staggered<2><<<1, 1, 0, st>>>((const uint32_t*)flag, (uint32_t*)echo, R, c.d); break;
      case 4: pp_staggered<4><<<1, 1, 0, st>>>((const uint32_t*)flag, (uint32_t*)echo, R, c.d); break;
      case 8: pp_staggered<8><<<1, 1, 0, st>>>((const uint32_t*)flag, (uint32_t*)echo, R, c.d); break;
    }
    usleep(1000);
    if (host_loop(flag, echo, R, lat, false)) return 1;
    cudaStreamSynchronize(st);
    char label[64];
    snprintf(label, sizeof label, "hostmem poll K=%d d=%uns", c.k, c.d);
    report(label, lat);
  }

  struct Cfg2 { int k; uint32_t d; } rc[] = {{2, 300}, {2, 500}, {4, 200}, {4, 300}, {8, 150}};
  for (auto c : rc) {
    memset(cells, 0, 4096);
    volatile uint32_t* ech = cells + 512;
    switch (c.k) {
      case 2: pp_replica<2><<<1, 1, 0, st>>>((const uint32_t*)cells, (uint32_t*)ech, R, c.d); break;
      case 4: pp_replica<4><<<1, 1, 0, st>>>((const uint32_t*)cells, (uint32_t*)ech, R, c.d); break;
      case 8: pp_replica<8><<<1, 1, 0, st>>>((const uint32_t*)cells, (uint32_t*)ech, R, c.d); break;
    }
    usleep(1000);
    lat.resize(R);
    bool bad = false;
    for (uint64_t r = 1; r <= R && !bad; ++r) {
      const uint64_t t0 = now_ns();
      for (int i = c.k - 1; i >= 0; --i) cells[32 * i] = uint32_t(r);
      const uint64_t dl = t0 + 2000000000ull;
      while (*ech != uint32_t(r)) { _mm_pause(); if (now_ns() > dl) { bad = true; break; } }
      lat[r - 1] = now_ns() - t0;
    }
    cudaStreamSynchronize(st);
    char label[64];
    snprintf(label, sizeof label, "replica lines K=%d d=%uns", c.k, c.d);
    if (!bad) report(label, lat); else printf("%s stalled\n", label);
  }
  struct Cfg3 { int w; uint32_t d; } wc[] = {{2, 600}, {4, 300}, {8, 150}, {16, 80}};
  for (auto c : wc) {
    memset(cells, 0, 4096);
    pp_warps<<<1, 32 * c.w, 0, st>>>((const uint32_t*)flag, (uint32_t*)echo, R, c.d);
    usleep(1000);
    if (host_loop(flag, echo, R, lat, false)) return 1;
    cudaStreamSynchronize(st);
    char label[64];
    snprintf(label, sizeof label, "staggered warps W=%d d=%uns", c.w, c.d);
    report(label, lat);
  }

  // C: dma-buf BAR1 mapping of device memory
  CUdevice dev;
  cuDeviceGet(&dev, 0);
  int dmabuf = 0;
  cuDeviceGetAttribute(&dmabuf, CU_DEVICE_ATTRIBUTE_DMA_BUF_SUPPORTED, dev);
  printf("DMA_BUF_SUPPORTED=%d  /dev/gdrdrv %s\n", dmabuf, access("/dev/gdrdrv", F_OK) == 0 ? "present" : "absent");
  CUdeviceptr dptr;
  const size_t sz = 2 << 20;
  CUresult cr = cuMemAlloc(&dptr, sz);
  printf("cuMemAlloc -> %d ptr=%#llx\n", int(cr), (unsigned long long)dptr);
  CUdeviceptr aligned = dptr;
  for (unsigned long long fl : {1ull, 0ull}) {
    int fd = -1;
    cr = cuMemGetHandleForAddressRange(&fd, aligned, sz, CU_MEM_RANGE_HANDLE_TYPE_DMA_BUF_FD, fl);
    printf("cuMemGetHandleForAddressRange(flags=%llu) -> %d fd=%d\n", fl, int(cr), fd);
    if (cr != CUDA_SUCCESS) continue;
    void* m = mmap(nullptr, sz, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    if (m == MAP_FAILED) {
      printf("  mmap(dma-buf) failed: %s\n", strerror(errno));
      close(fd);
      continue;
    }
    volatile uint32_t* hm = (volatile uint32_t*)m;
    hm[0] = 0xdeadbeef;
    _mm_sfence();
    uint32_t back = 0;
    cudaMemcpy(&back, (void*)aligned, 4, cudaMemcpyDeviceToHost);
    printf("  mmap ok; CPU wrote 0xdeadbeef, device reads %#x\n", back);
    for (int mode = 0; mode < 2; ++mode) {
      hm[0] = 0;
      memset(cells, 0, 4096);
      _mm_sfence();
      pp_devflag<<<1, 1, 0, st>>>((const uint32_t*)aligned, (uint32_t*)echo, R, mode);
      usleep(1000);
      if (host_loop(hm, echo, R, lat, true) == 0) report(mode ? "BAR1 devflag (volatile poll)" : "BAR1 devflag (relaxed.sys poll)", lat);
      cudaStreamSynchronize(st);
    }
    munmap(m, sz);
    close(fd);
    break;
  }
  return 0;
}
